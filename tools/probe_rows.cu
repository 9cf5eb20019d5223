// probe_rows.cu -- measurement probe (not product code): what makes writing
// CSR rows in a random row order slow on B200?  Synthetic rows (counts
// uniform in [80, 180], ~130 mean like cfg 5), N = 2^25 rows, random visit
// order.  Modes:
//   0 dense rows, random order            (the fill's situation)
//   1 rows padded to 8 ints (32-B sectors), random order
//   2 rows padded to 32 ints (128-B lines), random order
//   3 dense rows, sequential order
//   4 dense rows, random order, only the whole 32-B sectors of each row
//   5 dense rows, sequential order, only the partial sectors (edge pass)
//   6 dense rows, random order, whole sectors + edges to a side buffer
//     (64 B per row, full sectors), then the sequential edge pass
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_rows probe_rows.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include <algorithm>
#include <random>

__global__ void rows_kernel(const int64_t *__restrict__ off, const int32_t *__restrict__ ord, int64_t n,
                            int32_t *__restrict__ nbr, int mode, int4 *__restrict__ side) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = w0; t < n; t += nw) {
        const int64_t i = (mode == 3 || mode == 5) ? t : ord[t];
        const int64_t b = off[i], e = off[i + 1];
        if (mode == 4 || mode == 6) {
            const int64_t bs = (b + 7) & ~7ll, es = e & ~7ll;
            for (int64_t p = bs + lane; p < es; p += 32) nbr[p] = (int32_t)t;
            if (mode == 6 && lane < 4) side[4 * i + lane] = make_int4((int)t, (int)t, (int)t, (int)t);
        } else if (mode == 5) {
            const int64_t bs = min((int64_t)((b + 7) & ~7ll), e), es = max((int64_t)(e & ~7ll), bs);
            if (lane < bs - b) nbr[b + lane] = (int32_t)t;
            if (lane < e - es) nbr[es + lane] = (int32_t)t;
        } else {
            for (int64_t p = b + lane; p < e; p += 32) nbr[p] = (int32_t)t;
        }
    }
}

// sequential edge pass: one thread per row, reads its 64-B side record
__global__ void edge_kernel(const int64_t *__restrict__ off, int64_t n, int32_t *__restrict__ nbr,
                            const int4 *__restrict__ side) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t b = off[i], e = off[i + 1];
    const int64_t bs = min((int64_t)((b + 7) & ~7ll), e), es = max((int64_t)(e & ~7ll), bs);
    const int4 s0 = side[4 * i];
    for (int64_t p = b; p < bs; p++) nbr[p] = s0.x;
    for (int64_t p = es; p < e; p++) nbr[p] = s0.y;
}

int main() {
    const int64_t n = 1ll << 25;
    std::mt19937_64 g(1);
    std::vector<int64_t> cnt(n), off(n + 1), offp8(n + 1), offp32(n + 1);
    std::vector<int32_t> ord(n);
    off[0] = offp8[0] = offp32[0] = 0;
    for (int64_t i = 0; i < n; i++) {
        cnt[i] = 80 + (int64_t)(g() % 101);
        off[i + 1] = off[i] + cnt[i];
        offp8[i + 1] = offp8[i] + ((cnt[i] + 7) & ~7ll);
        offp32[i + 1] = offp32[i] + ((cnt[i] + 31) & ~31ll);
        ord[i] = (int32_t)i;
    }
    std::shuffle(ord.begin(), ord.end(), g);
    int64_t *d_off, *d_off8, *d_off32;
    int32_t *d_ord, *d_nbr;
    int4 *d_side;
    cudaMalloc(&d_off, (n + 1) * 8);
    cudaMalloc(&d_off8, (n + 1) * 8);
    cudaMalloc(&d_off32, (n + 1) * 8);
    cudaMalloc(&d_ord, n * 4);
    cudaMalloc(&d_side, n * 64);
    if (cudaMalloc(&d_nbr, offp32[n] * 4) != cudaSuccess) { printf("oom\n"); return 1; }
    cudaMemcpy(d_off, off.data(), (n + 1) * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d_off8, offp8.data(), (n + 1) * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d_off32, offp32.data(), (n + 1) * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d_ord, ord.data(), n * 4, cudaMemcpyHostToDevice);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char *names[] = {"dense_random", "pad8_random", "pad32_random", "dense_sequential",
                           "dense_random_whole_sectors_only", "dense_sequential_edges_only",
                           "dense_random_whole_sectors+side+edge_pass"};
    for (int mode = 0; mode < 7; mode++) {
        const int64_t *o = mode == 1 ? d_off8 : mode == 2 ? d_off32 : d_off;
        const int64_t bytes = (mode == 1 ? offp8[n] : mode == 2 ? offp32[n] : off[n]) * 4;
        auto go = [&]() {
            rows_kernel<<<sms * 8, 256>>>(o, d_ord, n, d_nbr, mode, d_side);
            if (mode == 6) edge_kernel<<<(unsigned)((n + 255) / 256), 256>>>(d_off, n, d_nbr, d_side);
        };
        go();
        cudaEventRecord(a);
        for (int r = 0; r < 5; r++) go();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 5;
        printf("{\"mode\": \"%s\", \"ms\": %.3f, \"row_bytes_GB\": %.3f, \"GBps\": %.1f}\n", names[mode], ms,
               bytes / 1e9, bytes / ms / 1e6);
    }
    cudaError_t err = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(err));
    return 0;
}
