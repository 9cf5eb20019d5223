// walk.cu -- FindNeighbors (Alg. 2) for all particles on the device.
//
// Work unit = up to 64 queries of one leaf bucket (the paper's "blocked
// approach", Sec. IV-E; particles are in tree order, so a unit's
// queries are spatial neighbours).  One warp per unit, persistent warps pull
// units from an atomic counter.  Per unit:
//   A10  descend from the root with Eq. 5 index ranges of the unit's query box
//        widened by R'_u = max_i R'_i (lemma L1/L2): empty cells
//        skipped, internal cells pushed on a per-warp stack (depth-first),
//        leaf cells culled by their tight bounding box (L3);
//   stage the surviving leaves' particles into shared memory, culled per
//        particle against the query box (Minkowski test, L3);
//   A11  test every query of the unit against the staged candidates with the
//        exact fp64 predicate ((dx*dx + dy*dy) + dz*dz) < (2h)^2 (no FMA:
//        __dmul_rn / __dadd_rn are never contracted); lanes = candidates,
//        __ballot_sync / __popc give the per-query count (count pass) or the
//        compacted write positions of the CSR row (fill pass, A13).
#include "common.cuh"
#include "scan.cuh"

namespace bt {

namespace {

constexpr int kQ = 64;          // queries per unit (== build.cu kUnitQ)
constexpr int kCand = 256;      // staged candidates per warp
constexpr int kWarpsPerBlock = 4;
constexpr int kWalkThreads = kWarpsPerBlock * 32;

struct WarpSmem {
    double qx[kQ], qy[kQ], qz[kQ], qT[kQ];
    int32_t qpos[kQ];
    int32_t qorig[kQ];
    double cx[kCand], cy[kCand], cz[kCand];
    int32_t cpos[kCand];
    int32_t corig[kCand];
    int32_t leafq[32];
};

struct WalkArgs {
    const double4 *rec;
    const double *h_tree;
    const NodeRec *nodes;
    const int32_t *cells;
    const int32_t *leaf_begin;
    const int32_t *leaf_count;
    const double *leaf_box;
    const int4 *units;
    int64_t n_units;
    double M;
    int root_is_leaf;
    int2 *stack;
    int64_t stack_per_warp;
    int32_t *counts;
    const int64_t *offsets;
    int32_t *nbr;
    unsigned long long *work;      // unit counter
    unsigned long long *stats;     // [0] staged, [1] tests
};

__device__ __forceinline__ double warp_min(double v) {
    for (int d = 16; d; d >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, d));
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
    for (int d = 16; d; d >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, d));
    return v;
}

// squared distance from point (x) to box [lo, hi], fp64, rounded ops
__device__ __forceinline__ double box_gap2(double x, double y, double z, const double *lo, const double *hi) {
    double gx = fmax(0.0, fmax(__dsub_rn(lo[0], x), __dsub_rn(x, hi[0])));
    double gy = fmax(0.0, fmax(__dsub_rn(lo[1], y), __dsub_rn(y, hi[1])));
    double gz = fmax(0.0, fmax(__dsub_rn(lo[2], z), __dsub_rn(z, hi[2])));
    return __dadd_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)), __dmul_rn(gz, gz));
}

template <bool FILL>
struct UnitState {
    int nq;
    int cnt0, cnt1;          // count pass: counts of queries lane, lane+32
    long long wr0, wr1;      // fill pass: next write slot of queries lane, lane+32
};

// Test all queries of the unit against the staged candidates [0, ncand).
template <bool FILL>
__device__ __forceinline__ void flush(WarpSmem &S, int ncand, UnitState<FILL> &st, int lane, int32_t *nbr) {
    const unsigned lt = lanemask_lt();
    for (int c0 = 0; c0 < ncand; c0 += 32) {
        int c = c0 + lane;
        bool valid = c < ncand;
        double x = valid ? S.cx[c] : 0.0, y = valid ? S.cy[c] : 0.0, z = valid ? S.cz[c] : 0.0;
        int32_t cp = valid ? S.cpos[c] : -1;
        int32_t co = valid ? S.corig[c] : 0;
        for (int q = 0; q < st.nq; q++) {
            double dx = __dsub_rn(S.qx[q], x);
            double dy = __dsub_rn(S.qy[q], y);
            double dz = __dsub_rn(S.qz[q], z);
            double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
            bool pass = valid && cp != S.qpos[q] && d2 < S.qT[q];
            unsigned m = __ballot_sync(0xffffffffu, pass);
            int pc = __popc(m);
            if (!FILL) {
                if (q < 32) { if (lane == q) st.cnt0 += pc; }
                else if (lane == q - 32) st.cnt1 += pc;
            } else {
                long long base = __shfl_sync(0xffffffffu, q < 32 ? st.wr0 : st.wr1, q & 31);
                if (pass) nbr[base + __popc(m & lt)] = co;
                if (q < 32) { if (lane == q) st.wr0 += pc; }
                else if (lane == q - 32) st.wr1 += pc;
            }
        }
    }
}

template <bool FILL>
__global__ void __launch_bounds__(kWalkThreads) walk_kernel(WalkArgs a) {
    __shared__ WarpSmem smem[kWarpsPerBlock];
    const int lane = threadIdx.x & 31;
    WarpSmem &S = smem[threadIdx.x >> 5];
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int2 *stk = a.stack + gwarp * a.stack_per_warp;
    const unsigned lt = lanemask_lt();
    unsigned long long staged = 0, tests = 0;

    for (;;) {
        unsigned long long u = 0;
        if (lane == 0) u = atomicAdd(a.work, 1ull);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= (unsigned long long)a.n_units) break;
        const int4 U = a.units[u];
        const int q0 = U.y;
        UnitState<FILL> st;
        st.nq = U.z;
        st.cnt0 = st.cnt1 = 0;
        st.wr0 = st.wr1 = 0;

        // ---- queries of the unit: coordinates, (2h)^2, R' and the query box
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        double Ru = 0.0;
        for (int k = lane; k < st.nq; k += 32) {
            int32_t p = q0 + k;
            double4 r = a.rec[p];
            double t = __dmul_rn(2.0, a.h_tree[p]);  // 2h (exact)
            S.qx[k] = r.x;
            S.qy[k] = r.y;
            S.qz[k] = r.z;
            S.qT[k] = __dmul_rn(t, t);
            S.qpos[k] = p;
            S.qorig[k] = (int32_t)__double_as_longlong(r.w);
            // R' = 2h (1 + 2^-40) + 2^-50 M   (lemma L1/L2)
            double Rp = __dadd_rn(__dmul_rn(t, 1.0 + 0x1p-40), __dmul_rn(0x1p-50, a.M));
            Ru = fmax(Ru, Rp);
            lo[0] = fmin(lo[0], r.x); lo[1] = fmin(lo[1], r.y); lo[2] = fmin(lo[2], r.z);
            hi[0] = fmax(hi[0], r.x); hi[1] = fmax(hi[1], r.y); hi[2] = fmax(hi[2], r.z);
        }
        for (int l = 0; l < 3; l++) { lo[l] = warp_min(lo[l]); hi[l] = warp_max(hi[l]); }
        Ru = warp_max(Ru);
        const double Ru2 = __dmul_rn(Ru, Ru);
        if (FILL) {
            if (lane < st.nq) st.wr0 = a.offsets[S.qorig[lane]];
            if (lane + 32 < st.nq) st.wr1 = a.offsets[S.qorig[lane + 32]];
        }
        __syncwarp();

        int ncand = 0;
        // stage one leaf's particles (per-particle cull against the query box)
        auto stage_leaf = [&](int32_t L) {
            const int32_t b0 = a.leaf_begin[L], m = a.leaf_count[L];
            for (int k0 = 0; k0 < m; k0 += 32) {
                if (ncand + 32 > kCand) {
                    __syncwarp();
                    flush<FILL>(S, ncand, st, lane, a.nbr);
                    tests += (unsigned long long)ncand * st.nq;
                    ncand = 0;
                    __syncwarp();
                }
                int k = k0 + lane;
                bool keep = false;
                double4 r;
                if (k < m) {
                    r = a.rec[b0 + k];
                    keep = box_gap2(r.x, r.y, r.z, lo, hi) < Ru2;
                }
                unsigned km = __ballot_sync(0xffffffffu, keep);
                if (keep) {
                    int slot = ncand + __popc(km & lt);
                    S.cx[slot] = r.x;
                    S.cy[slot] = r.y;
                    S.cz[slot] = r.z;
                    S.cpos[slot] = b0 + k;
                    S.corig[slot] = (int32_t)__double_as_longlong(r.w);
                }
                ncand += __popc(km);
                staged += (lane == 0) ? (unsigned long long)__popc(km) : 0ull;
            }
        };

        if (a.root_is_leaf) {
            stage_leaf(0);
        } else {
            // ---- A10: depth-first descent with Eq. 5 ranges
            int top = 1;
            if (lane == 0) stk[0] = make_int2(0, 0);
            __syncwarp();
            while (top > 0) {
                const int2 e = stk[top - 1];
                const NodeRec &nd = a.nodes[e.x];
                const int b = nd.b;
                int r0[3], r1[3];
                for (int l = 0; l < 3; l++) {
                    r0[l] = cell_coord(__dsub_rn(lo[l], Ru), nd.lo[l], nd.ext[l], b);
                    r1[l] = cell_coord(__dadd_rn(hi[l], Ru), nd.lo[l], nd.ext[l], b);
                }
                const long long nx = r1[0] - r0[0] + 1, ny = r1[1] - r0[1] + 1, nz = r1[2] - r0[2] + 1;
                const long long total = nx * ny * nz;
                const long long idx = (long long)e.y + lane;
                bool is_leaf = false, is_node = false;
                int32_t code = -1;
                if (idx < total) {
                    long long cx = r0[0] + idx % nx;
                    long long cy = r0[1] + (idx / nx) % ny;
                    long long cz = r0[2] + idx / (nx * ny);
                    long long j = cx + cy * b + cz * (long long)b * b;  // Eq. 3
                    code = a.cells[nd.cell_base + j];
                    if (code >= 0) {
                        // L3: cull the leaf if its tight box is farther than R'_u from the query box
                        const double *lb = a.leaf_box + 6 * (int64_t)code;
                        double gx = fmax(0.0, fmax(__dsub_rn(lb[0], hi[0]), __dsub_rn(lo[0], lb[3])));
                        double gy = fmax(0.0, fmax(__dsub_rn(lb[1], hi[1]), __dsub_rn(lo[1], lb[4])));
                        double gz = fmax(0.0, fmax(__dsub_rn(lb[2], hi[2]), __dsub_rn(lo[2], lb[5])));
                        double g2 = __dadd_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)), __dmul_rn(gz, gz));
                        is_leaf = g2 < Ru2;
                    } else if (code <= -2) {
                        is_node = true;
                    }
                }
                __syncwarp();
                const long long next = (long long)e.y + 32;
                if (next >= total) top--;
                else if (lane == 0) stk[top - 1].y = (int)next;
                unsigned nm = __ballot_sync(0xffffffffu, is_node);
                if (is_node) stk[top + __popc(nm & lt)] = make_int2(code_node(code), 0);
                top += __popc(nm);
                unsigned lm = __ballot_sync(0xffffffffu, is_leaf);
                if (is_leaf) S.leafq[__popc(lm & lt)] = code;
                __syncwarp();
                const int nl = __popc(lm);
                for (int i = 0; i < nl; i++) stage_leaf(S.leafq[i]);
                __syncwarp();
            }
        }
        __syncwarp();
        flush<FILL>(S, ncand, st, lane, a.nbr);
        tests += (unsigned long long)ncand * st.nq;
        if (!FILL) {
            if (lane < st.nq) a.counts[S.qorig[lane]] = st.cnt0;
            if (lane + 32 < st.nq) a.counts[S.qorig[lane + 32]] = st.cnt1;
        }
        __syncwarp();
    }
    if (!FILL && lane == 0) {
        atomicAdd(&a.stats[0], staged);
        atomicAdd(&a.stats[1], tests);
    }
}

// h in tree order + validation (h finite, > 0; |h| <= 1e150)
__global__ void gather_h_kernel(const double4 *__restrict__ rec, const double *__restrict__ h, int64_t n,
                                double *__restrict__ h_tree, int *bad) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        long long i = __double_as_longlong(rec[k].w);
        double v = h[i];
        if (!(v > 0.0 && v <= 1e150)) atomicOr(bad, 1);
        h_tree[k] = v;
    }
}

struct CountIn {
    const int32_t *c;
    __device__ long long operator()(int64_t i) const { return c[i]; }
};
struct OffsetOut {
    int64_t *off;
    unsigned long long *maxc;
    __device__ void operator()(int64_t i, long long exc, long long v) const {
        off[i] = exc;
        if (v > 0) atomicMax(maxc, (unsigned long long)v);
    }
};
__global__ void write_total_kernel(int64_t *off, int64_t n, const long long *total) { off[n] = *total; }

}  // namespace

void find_neighbors(TreeDev &t, const double *h, int32_t *counts, int64_t *offsets, int32_t *nbr_idx,
                    int64_t capacity, bool count_pass, bool fill_pass) {
    cudaStream_t st = stream();
    const int64_t n = t.n;
    if (n == 0) {
        if (offsets && count_pass) BT_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int64_t), st));
        t.total_pairs = t.max_count = t.staged = t.tests = t.exact_tests = 0;
        BT_CUDA(cudaStreamSynchronize(st));
        return;
    }
    const int sms = num_sms();
    DBuf<int> dbad(1);
    t.h_tree.reserve(n, 0);
    t.counters.reserve(8, 0);
    BT_CUDA(cudaMemsetAsync(dbad.p, 0, sizeof(int), st));
    BT_CUDA(cudaMemsetAsync(t.counters.p, 0, 8 * sizeof(int64_t), st));
    {
        Phase ph("search.gather_h");
        gather_h_kernel<<<grid_for(n, 256, (int64_t)sms * 16), 256, 0, st>>>(t.rec.p, h, n, t.h_tree.p, dbad.p);
        BT_LAUNCH("gather_h");
    }
    int hbad = 0;
    BT_CUDA(cudaMemcpyAsync(&hbad, dbad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    BT_CUDA(cudaStreamSynchronize(st));
    if (hbad) throw Error(BT_ERR_INPUT, "bt_find_neighbors: h must be finite, > 0 and <= 1e150");

    // persistent grid: all resident warps
    int per_sm = 0;
    BT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, walk_kernel<false>, kWalkThreads, 0));
    if (per_sm < 1) per_sm = 1;
    const unsigned grid = (unsigned)(sms * per_sm);
    const int64_t nwarps = (int64_t)grid * kWarpsPerBlock;
    t.stack_per_warp = 33 * (int64_t)(t.depth + 2);
    t.stack.reserve(nwarps * t.stack_per_warp, 0);

    WalkArgs a{};
    a.rec = t.rec.p;
    a.h_tree = t.h_tree.p;
    a.nodes = t.nodes.p;
    a.cells = t.cells.p;
    a.leaf_begin = t.leaf_begin.p;
    a.leaf_count = t.leaf_count.p;
    a.leaf_box = t.leaf_box.p;
    a.units = t.units.p;
    a.n_units = t.n_units;
    a.M = t.M;
    a.root_is_leaf = t.root_is_leaf ? 1 : 0;
    a.stack = t.stack.p;
    a.stack_per_warp = t.stack_per_warp;
    a.counts = counts;
    a.offsets = offsets;
    a.nbr = nbr_idx;
    a.work = (unsigned long long *)t.counters.p + 0;
    a.stats = (unsigned long long *)t.counters.p + 2;

    if (count_pass) {
        {
            Phase ph("search.count");
            walk_kernel<false><<<grid, kWalkThreads, 0, st>>>(a);
            BT_LAUNCH("walk_count");
        }
        DBuf<long long> dtot(1);
        {
            Phase ph("search.scan");
            device_scan<long long>(CountIn{counts}, OffsetOut{offsets, (unsigned long long *)t.counters.p + 5}, n,
                                   dtot.p);
            write_total_kernel<<<1, 1, 0, st>>>(offsets, n, dtot.p);
            BT_LAUNCH("write_total");
        }
    }
    int64_t hc[8];
    BT_CUDA(cudaMemcpyAsync(hc, t.counters.p, 8 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    int64_t total = 0;
    BT_CUDA(cudaMemcpyAsync(&total, offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    BT_CUDA(cudaStreamSynchronize(st));
    if (count_pass) {
        t.staged = hc[2];
        t.tests = hc[3];
        t.exact_tests = t.tests;
        t.max_count = hc[5];
    }
    t.total_pairs = total;
    if (!fill_pass || nbr_idx == nullptr) return;
    if (total > capacity)
        throw Error(BT_ERR_CAPACITY, "bt_find_neighbors: " + std::to_string(total) + " neighbor pairs exceed capacity " +
                                         std::to_string(capacity));
    BT_CUDA(cudaMemsetAsync(t.counters.p, 0, sizeof(int64_t), st));
    {
        Phase ph("search.fill");
        walk_kernel<true><<<grid, kWalkThreads, 0, st>>>(a);
        BT_LAUNCH("walk_fill");
    }
    BT_CUDA(cudaStreamSynchronize(st));
}

}  // namespace bt
