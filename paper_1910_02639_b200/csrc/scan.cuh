// scan.cuh -- device-wide exclusive prefix scan (three phases: tile reduce,
// scan of tile sums, tile scan + offset).  Generic over the value type T
// (any trivially copyable type with operator+ and a zero from T{}), an input
// functor in(i) -> T and an output functor out(i, exclusive_prefix, value).
// Used for the per-level cell scans (A6 in SURVEY 8(a)) and the count ->
// offset scan (A12).
#pragma once

#include "common.cuh"

namespace bt {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

template <class T>
__device__ __forceinline__ T shfl_up_t(T v, int d) {
    static_assert(sizeof(T) % 4 == 0, "scan value must be a multiple of 4 bytes");
    constexpr int W = sizeof(T) / 4;
    union U { T t; int w[W]; } u;
    u.t = v;
#pragma unroll
    for (int k = 0; k < W; k++) u.w[k] = __shfl_up_sync(0xffffffffu, u.w[k], d);
    return u.t;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive
// prefix and writes the block total.
template <class T>
__device__ __forceinline__ T block_exclusive(T v, T &total) {
    __shared__ T warp_tot[kScanThreads / kWarp];
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T o = shfl_up_t(inc, d);
        if (lane >= d) inc = inc + o;
    }
    if (lane == 31) warp_tot[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        T w = (lane < kScanThreads / kWarp) ? warp_tot[lane] : T{};
        T wi = w;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            T o = shfl_up_t(wi, d);
            if (lane >= d) wi = wi + o;
        }
        if (lane < kScanThreads / kWarp) warp_tot[lane] = wi;  // inclusive
    }
    __syncthreads();
    T base = wid ? warp_tot[wid - 1] : T{};
    total = warp_tot[kScanThreads / kWarp - 1];
    T exc = shfl_up_t(inc, 1);
    if (lane == 0) exc = T{};
    __syncthreads();
    return base + exc;
}

template <class T, class In>
__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(In in, int64_t n, T *tile_sums) {
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    T acc{};
#pragma unroll
    for (int k = 0; k < kScanItems; k++)
        if (base + k < n) acc = acc + in(base + k);
    T tot;
    block_exclusive(acc, tot);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

// single block: exclusive scan of tile sums in place, total to *total
template <class T>
__global__ void __launch_bounds__(kScanThreads) scan_tiles_kernel(T *tile_sums, int64_t ntiles, T *total) {
    T carry{};
    for (int64_t base = 0; base < ntiles; base += kScanThreads) {
        int64_t i = base + threadIdx.x;
        T v = (i < ntiles) ? tile_sums[i] : T{};
        T tot;
        T exc = block_exclusive(v, tot);
        if (i < ntiles) tile_sums[i] = carry + exc;
        carry = carry + tot;
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

template <class T, class In, class Out>
__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(In in, Out out, int64_t n, const T *tile_offsets) {
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    T vals[kScanItems];
    T acc{};
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        vals[k] = (base + k < n) ? in(base + k) : T{};
        acc = acc + vals[k];
    }
    T tot;
    T pre = tile_offsets[blockIdx.x] + block_exclusive(acc, tot);
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        if (base + k < n) out(base + k, pre, vals[k]);
        pre = pre + vals[k];
    }
}

// in-place exclusive scan of an array of tile sums (the recursive level)
template <class T>
struct TileIn {
    const T *p;
    __device__ T operator()(int64_t i) const { return p[i]; }
};
template <class T>
struct TileOut {
    T *p;
    __device__ void operator()(int64_t i, const T &exc, const T &) const { p[i] = exc; }
};

// one tile (n <= kScanTile): the whole scan in one block, one launch
template <class T, class In, class Out>
__global__ void __launch_bounds__(kScanThreads) scan_single_kernel(In in, Out out, int64_t n, T *total) {
    const int64_t base = (int64_t)threadIdx.x * kScanItems;
    T vals[kScanItems];
    T acc{};
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        vals[k] = (base + k < n) ? in(base + k) : T{};
        acc = acc + vals[k];
    }
    T tot;
    T pre = block_exclusive(acc, tot);
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        if (base + k < n) out(base + k, pre, vals[k]);
        pre = pre + vals[k];
    }
    if (threadIdx.x == 0 && total) *total = tot;
}

// Exclusive scan of n items; total (device pointer, may be null) receives the sum.
template <class T, class In, class Out>
void device_scan(In in, Out out, int64_t n, T *total) {
    int64_t ntiles = (n + kScanTile - 1) / kScanTile;
    if (ntiles <= 1) {
        scan_single_kernel<T, In, Out><<<1, kScanThreads, 0, stream()>>>(in, out, n, total);
        BT_LAUNCH("scan_single");
        return;
    }
    DBuf<T> tiles(ntiles);
    scan_reduce_kernel<T, In><<<(unsigned)ntiles, kScanThreads, 0, stream()>>>(in, n, tiles.p);
    BT_LAUNCH("scan_reduce");
    if (ntiles > kScanTile) {  // many tiles: scan the tile sums in parallel, not in one block
        device_scan<T>(TileIn<T>{tiles.p}, TileOut<T>{tiles.p}, ntiles, total);
    } else {
        scan_tiles_kernel<T><<<1, kScanThreads, 0, stream()>>>(tiles.p, ntiles, total);
        BT_LAUNCH("scan_tiles");
    }
    scan_apply_kernel<T, In, Out><<<(unsigned)ntiles, kScanThreads, 0, stream()>>>(in, out, n, tiles.p);
    BT_LAUNCH("scan_apply");
}

}  // namespace bt
