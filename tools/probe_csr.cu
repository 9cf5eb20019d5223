// probe_csr.cu -- measurement probe (not product code): the cost of writing a
// CSR of the fill's shape.  One warp per row writes counts[i] 4-byte entries
// at nbr[offsets[i] ..] with coalesced stores; rows visited in tree order
// (row i = perm[t], t = 0, 1, ...: the order the fill meets them) or in caller
// order (i = t: sequential).  Times with CUDA events; returns ms.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void rows_kernel(const int64_t *__restrict__ off, const int32_t *__restrict__ perm, int64_t n,
                            int32_t *__restrict__ nbr, int mode) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = w0; t < n; t += nw) {
        const int64_t i = mode == 0 ? perm[t] : t;
        const int64_t b = off[i], e = off[i + 1];
        for (int64_t p = b + lane; p < e; p += 32) nbr[p] = (int32_t)t;
    }
}

// rows in tree order, the row bounds of 32 rows loaded at once (lanes = rows),
// then each row written by the whole warp: no dependent-load chain per row
__global__ void rows_batched_kernel(const int64_t *__restrict__ off, const int32_t *__restrict__ perm, int64_t n,
                                    int32_t *__restrict__ nbr) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t0 = 32 * w0; t0 < n; t0 += 32 * nw) {
        int64_t b = 0, e = 0;
        if (t0 + lane < n) {
            const int64_t i = perm[t0 + lane];
            b = off[i];
            e = off[i + 1];
        }
        for (int r = 0; r < 32; r++) {
            const int64_t rb = __shfl_sync(0xffffffffu, b, r), re = __shfl_sync(0xffffffffu, e, r);
            for (int64_t p = rb + lane; p < re; p += 32) nbr[p] = (int32_t)(t0 + r);
        }
    }
}

extern "C" float probe_rows(const int64_t *off, const int32_t *perm, int64_t n, int32_t *nbr, int mode, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto go = [&]() {
        if (mode == 2) rows_batched_kernel<<<sms * 8, 256>>>(off, perm, n, nbr);
        else rows_kernel<<<sms * 8, 256>>>(off, perm, n, nbr, mode);
    };
    go();
    cudaEventRecord(a);
    for (int r = 0; r < reps; r++) go();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}
