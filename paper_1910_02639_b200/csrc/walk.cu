// walk.cu -- FindNeighbors (Alg. 2) for all particles on the device.
//
// Work unit = up to 64 queries of one leaf bucket (the paper's "blocked
// approach", Sec. IV-E: particles are in tree order, so a unit's queries
// are spatial neighbours).  One warp per unit; persistent warps pull units
// from an atomic counter.
//
// Test pass (count), per unit:
//   A10  descend from the root with Eq. 5 index ranges of the unit's query box
//        widened by R'_u = max_i R'_i (lemma L1/L2): empty cells
//        skipped, internal cells pushed on a per-warp stack (depth first),
//        leaf cells culled by their tight bounding box (L3);
//        stage the surviving leaves' particles into shared memory, culled per
//        particle against the query box in fp64 (Minkowski test, L3), as fp32
//        coordinates relative to the unit centre;
//   A11  lanes = candidates (two per lane, packed f32x2), loop over queries:
//        s32 = fp32 squared distance; s32 < A_i -> certainly a neighbor,
//        s32 >= B_i -> certainly not, else the exact fp64 predicate
//        ((dx*dx + dy*dy) + dz*dz) < (2h)^2 decides (lemma L4 gives A_i, B_i
//        from the error bound of the fp32 evaluation):
//        the recorded neighbor set is exactly the fp64 one.
//        __ballot_sync gives the per-(query, 64-candidate chunk) neighbor
//        masks; their __popc sums are the counts.  The masks and the chunk's
//        candidate indices are recorded in an arena.
// Scan (A12): offsets = exclusive scan of counts.
// Fill pass (A13): replay the recorded masks: __popc(mask & lanemask_lt)
//        gives each neighbor's slot in its CSR row; coalesced row writes.
#include <algorithm>
#include <cfloat>

#include "common.cuh"
#include "scan.cuh"

namespace bt {

namespace {

constexpr int kQ = 64;          // queries per unit (== build.cu kUnitQ)
constexpr int kCand = 256;      // staged candidates per warp and batch
constexpr int kWarpsPerBlock = 4;
constexpr int kWalkThreads = kWarpsPerBlock * 32;

// device counters (int64 slots of TreeDev::counters)
enum {
    C_WORK = 0,      // unit counter (test pass)
    C_MASK = 1,      // mask words requested
    C_CAND = 2,      // candidate slots requested
    C_BATCH = 3,     // batches requested
    C_STAGED = 4,
    C_TESTS = 5,
    C_EXACT = 6,
    C_MAXC = 7,
    C_WORK2 = 8,     // unit counter (fill pass)
    C_HSUM = 9,      // checksum of h (bit patterns)
    C_N = 16
};

using Batch = WalkBatch;

struct WarpSmem {
    float4 q0[kQ];              // ax, ax, ay, ay   (fp32, relative to the unit centre)
    float4 q1[kQ];              // az, az, A, B     (certain-accept / certain-reject thresholds)
    double qx[kQ], qy[kQ], qz[kQ], qT[kQ];  // fp64 query data for the exact band
    int32_t qpos[kQ];
    int32_t qorig[kQ];
    int32_t qself[kQ];          // batch-local slot of the query itself, -1 if not in this batch
    float2 px[kCand / 2], py[kCand / 2], pz[kCand / 2];  // chunk k, lane l: (c[64k+l], c[64k+32+l])
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
    int exact_only;
    int2 *stack;
    int64_t stack_per_warp;
    int32_t *counts;
    const int64_t *offsets;
    int32_t *nbr;
    long long *ctr;
    // arena
    unsigned long long *masks;
    long long mask_cap;
    int32_t *cands;
    long long cand_cap;
    Batch *batches;
    long long batch_cap;
    int32_t *head;  // first batch of each unit
};

__device__ __forceinline__ double warp_min(double v) {
    for (int d = 16; d; d >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, d));
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
    for (int d = 16; d; d >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, d));
    return v;
}

// packed fp32 pair arithmetic (sm_100a FADD2 / FMUL2 / FFMA2)
__device__ __forceinline__ unsigned long long f2(float2 v) {
    return ((unsigned long long)__float_as_uint(v.y) << 32) | __float_as_uint(v.x);
}
__device__ __forceinline__ unsigned long long f2_sub(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// Exact predicate (the definition): ((dx*dx + dy*dy) + dz*dz) < T, fp64, no FMA.
__device__ __forceinline__ bool exact_pair(double qx, double qy, double qz, double T, const double4 &c) {
    double dx = __dsub_rn(qx, c.x), dy = __dsub_rn(qy, c.y), dz = __dsub_rn(qz, c.z);
    double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    return d2 < T;
}

// Lemma L4: thresholds A <= B (fp32) such that for the
// fp32 squared distance s32 of a pair whose coordinates relative to the unit
// centre are bounded by E (per axis),
//   s32 <  A  =>  fp64 predicate true,     s32 >= B  =>  fp64 predicate false.
// All slack factors round the bounds outward.
__device__ __forceinline__ void l4_thresholds(double T, double E, bool exact_only, float &A, float &B) {
    const double u = 0x1p-53, w = 0x1p-24;
    if (exact_only || !(E < 1e15)) {
        A = 0.0f;
        B = __int_as_float(0x7f800000);  // +inf: every pair goes to the fp64 predicate
        return;
    }
    const double eps = u * E + w * (1.0 + u) * E + 0x1p-149;  // |a - (x - c)| per coordinate
    const double a0 = 2.0 * eps * (1.0 + w) + 0x1p-150;        // |d - D| = a0 + w |D|
    const double g3 = 3.0 * w / (1.0 - 3.0 * w);
    auto err = [&](double S) {
        double D = 3.0 * a0 * a0 + 2.0 * 1.7320508075688775 * a0 * (1.0 + w) * sqrt(S) + (2.0 * w + w * w) * S;
        return (D + g3 * (S + D) + 3.0 * 0x1p-150) * 1.0001;
    };
    const double Tm = T * (1.0 - 8.0 * u);  // <= T / (1 + gamma_5)
    const double Tp = T * (1.0 + 8.0 * u);  // >= T / (1 - gamma_5)
    A = 0.0f;
    if (a0 <= 0.01 * sqrt(Tm)) {  // S - err(S) increasing on [Tm, inf)
        double g = (Tm - err(Tm)) * (1.0 - 0x1p-40);
        if (g > 0.0) A = __double2float_rd(g);
    }
    double hb = (Tp + err(Tp)) * (1.0 + 0x1p-40);
    B = (hb < 3.0e38) ? __double2float_ru(hb) : __int_as_float(0x7f800000);
}

// squared distance from point to box [lo, hi], fp64 rounded ops
__device__ __forceinline__ double box_gap2(double x, double y, double z, const double *lo, const double *hi) {
    double gx = fmax(0.0, fmax(__dsub_rn(lo[0], x), __dsub_rn(x, hi[0])));
    double gy = fmax(0.0, fmax(__dsub_rn(lo[1], y), __dsub_rn(y, hi[1])));
    double gz = fmax(0.0, fmax(__dsub_rn(lo[2], z), __dsub_rn(z, hi[2])));
    return __dadd_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)), __dmul_rn(gz, gz));
}

// ---------------------------------------------------------------------------
// Test pass
// ---------------------------------------------------------------------------
struct CountState {
    int nq;
    int c0, c1;           // counts of queries lane, lane + 32
    int prev_batch;
    long long tests, exact;
};

// Test all queries of the unit against the staged batch [0, ncand), record
// masks and candidates, accumulate counts.
__device__ __noinline__ void test_batch(WarpSmem &S, int ncand, CountState &st, int lane, const WalkArgs &a,
                                        int64_t unit) {
    const int nch = (ncand + 63) >> 6;
    const float inf = __int_as_float(0x7f800000);
    // pad the last chunk with +inf coordinates (s32 = +inf: never a neighbor)
    for (int c = ncand + lane; c < nch * 64; c += 32) {
        int k = c >> 6, l = c & 31, hi = (c >> 5) & 1;
        float *px = reinterpret_cast<float *>(&S.px[32 * k + l]);
        float *py = reinterpret_cast<float *>(&S.py[32 * k + l]);
        float *pz = reinterpret_cast<float *>(&S.pz[32 * k + l]);
        px[hi] = inf;
        py[hi] = inf;
        pz[hi] = inf;
        S.corig[c] = -1;
        S.cpos[c] = -1;
    }
    // arena allocation for this batch
    long long mb = 0, cb = 0, bi = 0;
    if (lane == 0) {
        mb = atomicAdd((unsigned long long *)&a.ctr[C_MASK], (unsigned long long)(nch * st.nq));
        cb = atomicAdd((unsigned long long *)&a.ctr[C_CAND], (unsigned long long)(nch * 64));
        bi = atomicAdd((unsigned long long *)&a.ctr[C_BATCH], 1ull);
    }
    mb = __shfl_sync(0xffffffffu, mb, 0);
    cb = __shfl_sync(0xffffffffu, cb, 0);
    bi = __shfl_sync(0xffffffffu, bi, 0);
    const bool record = (mb + (long long)nch * st.nq <= a.mask_cap) && (cb + (long long)nch * 64 <= a.cand_cap) &&
                        (bi < a.batch_cap);
    __syncwarp();
    if (record) {
        for (int c = lane; c < nch * 64; c += 32) a.cands[cb + c] = S.corig[c];
        if (lane == 0) {
            a.batches[bi] = Batch{mb, cb, ncand, -1};
            if (st.prev_batch >= 0) a.batches[st.prev_batch].next = (int)bi;
            else a.head[unit] = (int)bi;
        }
        st.prev_batch = (int)bi;
    }
    for (int k = 0; k < nch; k++) {
        const unsigned long long cx = f2(S.px[32 * k + lane]);
        const unsigned long long cy = f2(S.py[32 * k + lane]);
        const unsigned long long cz = f2(S.pz[32 * k + lane]);
        const int cp0 = S.cpos[64 * k + lane], cp1 = S.cpos[64 * k + 32 + lane];
        for (int q = 0; q < st.nq; q++) {
            const float4 Q0 = S.q0[q], Q1 = S.q1[q];
            unsigned long long dx = f2_sub(cx, f2(make_float2(Q0.x, Q0.y)));
            unsigned long long dy = f2_sub(cy, f2(make_float2(Q0.z, Q0.w)));
            unsigned long long dz = f2_sub(cz, f2(make_float2(Q1.x, Q1.y)));
            unsigned long long s = f2_mul(dx, dx);
            s = f2_fma(dy, dy, s);
            s = f2_fma(dz, dz, s);
            const float s0 = __uint_as_float((unsigned)s), s1 = __uint_as_float((unsigned)(s >> 32));
            const bool a0 = s0 < Q1.z, a1 = s1 < Q1.z;
            const bool u0 = !a0 && s0 < Q1.w, u1 = !a1 && s1 < Q1.w;
            unsigned m0 = __ballot_sync(0xffffffffu, a0);
            unsigned m1 = __ballot_sync(0xffffffffu, a1);
            if (__any_sync(0xffffffffu, u0 || u1)) {
                // exact band: the fp64 predicate decides (rare)
                const double qx = S.qx[q], qy = S.qy[q], qz = S.qz[q], T = S.qT[q];
                const int qp = S.qpos[q];
                bool e0 = false, e1 = false;
                if (u0) e0 = cp0 != qp && exact_pair(qx, qy, qz, T, a.rec[cp0]);
                if (u1) e1 = cp1 != qp && exact_pair(qx, qy, qz, T, a.rec[cp1]);
                m0 |= __ballot_sync(0xffffffffu, e0);
                m1 |= __ballot_sync(0xffffffffu, e1);
                st.exact += __popc(__ballot_sync(0xffffffffu, u0)) + __popc(__ballot_sync(0xffffffffu, u1));
            }
            // self is never its own neighbor (R12)
            const int sl = S.qself[q] - 64 * k;
            if ((unsigned)sl < 64u) {
                if (sl < 32) m0 &= ~(1u << sl);
                else m1 &= ~(1u << (sl - 32));
            }
            const int pc = __popc(m0) + __popc(m1);
            if (q < 32) st.c0 += (lane == q) ? pc : 0;
            else st.c1 += (lane == q - 32) ? pc : 0;
            if (record && lane == 0) a.masks[mb + (long long)k * st.nq + q] = ((unsigned long long)m1 << 32) | m0;
        }
    }
    st.tests += (long long)ncand * st.nq;
}

__global__ void __launch_bounds__(kWalkThreads) test_kernel(WalkArgs a) {
    __shared__ WarpSmem smem[kWarpsPerBlock];
    const int lane = threadIdx.x & 31;
    WarpSmem &S = smem[threadIdx.x >> 5];
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int2 *stk = a.stack + gwarp * a.stack_per_warp;
    const unsigned lt = lanemask_lt();
    long long staged = 0, tests = 0, exact = 0;

    for (;;) {
        unsigned long long u = 0;
        if (lane == 0) u = atomicAdd((unsigned long long *)&a.ctr[C_WORK], 1ull);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= (unsigned long long)a.n_units) break;
        const int4 U = a.units[u];
        const int q0 = U.y;
        CountState st;
        st.nq = U.z;
        st.c0 = st.c1 = 0;
        st.prev_batch = -1;
        st.tests = st.exact = 0;
        if (lane == 0) a.head[u] = -1;

        // ---- query box, R'_u
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
            S.qself[k] = -1;
            // R' = 2h (1 + 2^-40) + 2^-50 M   (lemma L1/L2)
            double Rp = __dadd_rn(__dmul_rn(t, 1.0 + 0x1p-40), __dmul_rn(0x1p-50, a.M));
            Ru = fmax(Ru, Rp);
            lo[0] = fmin(lo[0], r.x); lo[1] = fmin(lo[1], r.y); lo[2] = fmin(lo[2], r.z);
            hi[0] = fmax(hi[0], r.x); hi[1] = fmax(hi[1], r.y); hi[2] = fmax(hi[2], r.z);
        }
        for (int l = 0; l < 3; l++) { lo[l] = warp_min(lo[l]); hi[l] = warp_max(hi[l]); }
        Ru = warp_max(Ru);
        const double Ru2 = __dmul_rn(Ru, Ru);
        // unit centre c and the a-priori coordinate bound E (|x - c| <= E per
        // axis for every query and every staged candidate)
        double c[3], E = 0.0, Mu = 0.0;
        for (int l = 0; l < 3; l++) {
            c[l] = 0.5 * (lo[l] + hi[l]);
            E = fmax(E, 0.5 * (hi[l] - lo[l]));
            Mu = fmax(Mu, fmax(fabs(lo[l]), fabs(hi[l])));
        }
        E = (E + Ru) * 1.0001 + 4.0 * 0x1p-53 * Mu;
        for (int k = lane; k < st.nq; k += 32) {
            float ax = __double2float_rn(__dsub_rn(S.qx[k], c[0]));
            float ay = __double2float_rn(__dsub_rn(S.qy[k], c[1]));
            float az = __double2float_rn(__dsub_rn(S.qz[k], c[2]));
            float A, B;
            l4_thresholds(S.qT[k], E, a.exact_only != 0, A, B);
            S.q0[k] = make_float4(ax, ax, ay, ay);
            S.q1[k] = make_float4(az, az, A, B);
        }
        __syncwarp();

        int ncand = 0;
        auto stage_leaf = [&](int32_t L) {
            const int32_t b0 = a.leaf_begin[L], m = a.leaf_count[L];
            for (int k0 = 0; k0 < m; k0 += 32) {
                if (ncand + 32 > kCand) {
                    __syncwarp();
                    test_batch(S, ncand, st, lane, a, (int64_t)u);
                    for (int k = lane; k < st.nq; k += 32) S.qself[k] = -1;
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
                    int ck = slot >> 6, cl = slot & 31, ch = (slot >> 5) & 1;
                    reinterpret_cast<float *>(&S.px[32 * ck + cl])[ch] = __double2float_rn(__dsub_rn(r.x, c[0]));
                    reinterpret_cast<float *>(&S.py[32 * ck + cl])[ch] = __double2float_rn(__dsub_rn(r.y, c[1]));
                    reinterpret_cast<float *>(&S.pz[32 * ck + cl])[ch] = __double2float_rn(__dsub_rn(r.z, c[2]));
                    S.cpos[slot] = b0 + k;
                    S.corig[slot] = (int32_t)__double_as_longlong(r.w);
                    const int qi = b0 + k - q0;
                    if (qi >= 0 && qi < st.nq) S.qself[qi] = slot;
                }
                ncand += __popc(km);
                staged += (lane == 0) ? __popc(km) : 0;
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
        if (ncand > 0 || st.prev_batch < 0) test_batch(S, ncand, st, lane, a, (int64_t)u);
        if (lane < st.nq) a.counts[S.qorig[lane]] = st.c0;
        if (lane + 32 < st.nq) a.counts[S.qorig[lane + 32]] = st.c1;
        tests += st.tests;
        exact += st.exact;
        __syncwarp();
    }
    if (lane == 0) {
        atomicAdd((unsigned long long *)&a.ctr[C_STAGED], (unsigned long long)staged);
        atomicAdd((unsigned long long *)&a.ctr[C_TESTS], (unsigned long long)tests);
        atomicAdd((unsigned long long *)&a.ctr[C_EXACT], (unsigned long long)exact);
    }
}

// ---------------------------------------------------------------------------
// Fill pass: replay the recorded masks into the CSR rows
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kWalkThreads) fill_kernel(WalkArgs a) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
    for (;;) {
        unsigned long long u = 0;
        if (lane == 0) u = atomicAdd((unsigned long long *)&a.ctr[C_WORK2], 1ull);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= (unsigned long long)a.n_units) break;
        const int4 U = a.units[u];
        const int nq = U.z;
        long long wr0 = 0, wr1 = 0;
        if (lane < nq) wr0 = a.offsets[(int32_t)__double_as_longlong(a.rec[U.y + lane].w)];
        if (lane + 32 < nq) wr1 = a.offsets[(int32_t)__double_as_longlong(a.rec[U.y + lane + 32].w)];
        for (int b = a.head[u]; b >= 0;) {
            const Batch B = a.batches[b];
            const int nch = (B.ncand + 63) >> 6;
            for (int k = 0; k < nch; k++) {
                const int32_t c0 = a.cands[B.cand_base + 64 * k + lane];
                const int32_t c1 = a.cands[B.cand_base + 64 * k + 32 + lane];
                const unsigned long long *mk = a.masks + B.mask_base + (long long)k * nq;
                const unsigned long long mA = (lane < nq) ? mk[lane] : 0ull;
                const unsigned long long mB = (lane + 32 < nq) ? mk[lane + 32] : 0ull;
                for (int q = 0; q < nq; q++) {
                    const unsigned long long m = __shfl_sync(0xffffffffu, q < 32 ? mA : mB, q & 31);
                    if (m == 0ull) continue;
                    const long long base = __shfl_sync(0xffffffffu, q < 32 ? wr0 : wr1, q & 31);
                    const unsigned lo = (unsigned)m, hi = (unsigned)(m >> 32);
                    const int plo = __popc(lo);
                    if ((lo >> lane) & 1u) a.nbr[base + __popc(lo & lt)] = c0;
                    if ((hi >> lane) & 1u) a.nbr[base + plo + __popc(hi & lt)] = c1;
                    const int pc = plo + __popc(hi);
                    if (q < 32) wr0 += (lane == q) ? pc : 0;
                    else wr1 += (lane == q - 32) ? pc : 0;
                }
            }
            b = B.next;
        }
    }
}

// h in tree order + validation (h finite, > 0, <= 1e150) + checksum of h
__global__ void gather_h_kernel(const double4 *__restrict__ rec, const double *__restrict__ h, int64_t n,
                                double *__restrict__ h_tree, int *bad, long long *hsum) {
    long long acc = 0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        long long i = __double_as_longlong(rec[k].w);
        double v = h[i];
        if (!(v > 0.0 && v <= 1e150)) atomicOr(bad, 1);
        h_tree[k] = v;
        acc += __double_as_longlong(v) * (2 * i + 1);
    }
    for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
    if ((threadIdx.x & 31) == 0) atomicAdd((unsigned long long *)hsum, (unsigned long long)acc);
}

struct CountIn {
    const int32_t *c;
    __device__ long long operator()(int64_t i) const { return c[i]; }
};
struct OffsetOut {
    int64_t *off;
    __device__ void operator()(int64_t i, long long exc, long long) const { off[i] = exc; }
};
__global__ void write_total_kernel(int64_t *off, int64_t n, const long long *total) { off[n] = *total; }

__global__ void max_count_kernel(const int32_t *c, int64_t n, long long *out) {
    int m = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, c[i]);
    for (int d = 16; d; d >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, d));
    if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long *)out, (unsigned long long)m);
}

thread_local int g_exact_only = 0;

}  // namespace

void set_exact_only(int on) { g_exact_only = on; }

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
    t.counters.reserve(C_N, 0);
    BT_CUDA(cudaMemsetAsync(dbad.p, 0, sizeof(int), st));
    BT_CUDA(cudaMemsetAsync(t.counters.p + C_HSUM, 0, sizeof(int64_t), st));
    {
        Phase ph("search.gather_h");
        gather_h_kernel<<<grid_for(n, 256, (int64_t)sms * 16), 256, 0, st>>>(t.rec.p, h, n, t.h_tree.p, dbad.p,
                                                                            (long long *)t.counters.p + C_HSUM);
        BT_LAUNCH("gather_h");
    }
    int hbad = 0;
    long long hsum = 0;
    BT_CUDA(cudaMemcpyAsync(&hbad, dbad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    BT_CUDA(cudaMemcpyAsync(&hsum, t.counters.p + C_HSUM, sizeof(long long), cudaMemcpyDeviceToHost, st));
    BT_CUDA(cudaStreamSynchronize(st));
    if (hbad) throw Error(BT_ERR_INPUT, "bt_find_neighbors: h must be finite, > 0 and <= 1e150");

    // persistent grid: all resident warps
    int per_sm = 0;
    BT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, test_kernel, kWalkThreads, 0));
    if (per_sm < 1) per_sm = 1;
    const unsigned grid = (unsigned)(sms * per_sm);
    const int64_t nwarps = (int64_t)grid * kWarpsPerBlock;
    t.stack_per_warp = 33 * (int64_t)(t.depth + 2);
    t.stack.reserve(nwarps * t.stack_per_warp, 0);
    t.head.reserve(t.n_units, 0);

    // the recorded masks of a previous test pass are reused by a fill-only
    // call when the tree, h pointer, exactness mode and h checksum all match
    const bool have_record = t.rec_valid && t.rec_h == h && t.rec_hsum == hsum && t.rec_exact == g_exact_only;
    const bool run_test = count_pass || !have_record;

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
    a.exact_only = g_exact_only;
    a.stack = t.stack.p;
    a.stack_per_warp = t.stack_per_warp;
    a.offsets = offsets;
    a.nbr = nbr_idx;
    a.ctr = (long long *)t.counters.p;
    a.head = t.head.p;

    DBuf<int32_t> tmp_counts;
    if (run_test) {
        int32_t *cnt = counts;
        if (!cnt) {
            tmp_counts.alloc(n);
            cnt = tmp_counts.p;
        }
        a.counts = cnt;
        // arena sized from the previous run on this thread (grown on overflow)
        static thread_local double mask_per_q = 12.0, cand_per_q = 24.0, batch_per_unit = 1.5;
        for (int attempt = 0;; attempt++) {
            long long mcap = (long long)(mask_per_q * n) + 4096, ccap = (long long)(cand_per_q * n) + 4096;
            long long bcap = (long long)(batch_per_unit * t.n_units) + 1024;
            t.arena_masks.reserve(mcap, 0);
            t.arena_cands.reserve(ccap, 0);
            t.arena_batches.reserve(bcap, 0);
            a.masks = t.arena_masks.p;
            a.mask_cap = (long long)t.arena_masks.n;
            a.cands = t.arena_cands.p;
            a.cand_cap = (long long)t.arena_cands.n;
            a.batches = t.arena_batches.p;
            a.batch_cap = (long long)t.arena_batches.n;
            BT_CUDA(cudaMemsetAsync(t.counters.p, 0, C_HSUM * sizeof(int64_t), st));
            {
                Phase ph("search.count");
                test_kernel<<<grid, kWalkThreads, 0, st>>>(a);
                BT_LAUNCH("walk_test");
            }
            long long hc[C_N];
            BT_CUDA(cudaMemcpyAsync(hc, t.counters.p, C_N * sizeof(long long), cudaMemcpyDeviceToHost, st));
            BT_CUDA(cudaStreamSynchronize(st));
            t.staged = hc[C_STAGED];
            t.tests = hc[C_TESTS];
            t.exact_tests = hc[C_EXACT];
            const bool fits = hc[C_MASK] <= a.mask_cap && hc[C_CAND] <= a.cand_cap && hc[C_BATCH] <= a.batch_cap;
            mask_per_q = std::max(mask_per_q, 1.1 * (double)hc[C_MASK] / (double)n);
            cand_per_q = std::max(cand_per_q, 1.1 * (double)hc[C_CAND] / (double)n);
            batch_per_unit = std::max(batch_per_unit, 1.1 * (double)hc[C_BATCH] / (double)std::max<int64_t>(1, t.n_units));
            if (fits || !fill_pass || nbr_idx == nullptr) {
                t.rec_valid = fits;
                t.rec_h = h;
                t.rec_hsum = hsum;
                t.rec_exact = g_exact_only;
                break;
            }
            // arena overflow with a fill to do: grow and repeat the test pass
            if (attempt > 2) throw Error(BT_ERR_OOM, "bt_find_neighbors: candidate arena does not converge");
        }
        if (count_pass) {
            DBuf<long long> dtot(1);
            Phase ph("search.scan");
            device_scan<long long>(CountIn{cnt}, OffsetOut{offsets}, n, dtot.p);
            write_total_kernel<<<1, 1, 0, st>>>(offsets, n, dtot.p);
            BT_LAUNCH("write_total");
            BT_CUDA(cudaMemsetAsync(t.counters.p + C_MAXC, 0, sizeof(int64_t), st));
            max_count_kernel<<<grid_for(n, 256, (int64_t)sms * 8), 256, 0, st>>>(cnt, n,
                                                                                  (long long *)t.counters.p + C_MAXC);
            BT_LAUNCH("max_count");
        }
    }
    int64_t total = 0, maxc = 0;
    BT_CUDA(cudaMemcpyAsync(&total, offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    if (count_pass) BT_CUDA(cudaMemcpyAsync(&maxc, t.counters.p + C_MAXC, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    BT_CUDA(cudaStreamSynchronize(st));
    if (count_pass) t.max_count = maxc;
    t.total_pairs = total;
    if (!fill_pass || nbr_idx == nullptr) return;
    if (total > capacity)
        throw Error(BT_ERR_CAPACITY, "bt_find_neighbors: " + std::to_string(total) + " neighbor pairs exceed capacity " +
                                         std::to_string(capacity));
    if (!t.rec_valid) throw Error(BT_ERR_CUDA, "bt_find_neighbors: internal: no recorded test pass");
    a.masks = t.arena_masks.p;
    a.cands = t.arena_cands.p;
    a.batches = t.arena_batches.p;
    BT_CUDA(cudaMemsetAsync(t.counters.p + C_WORK2, 0, sizeof(int64_t), st));
    {
        Phase ph("search.fill");
        fill_kernel<<<grid, kWalkThreads, 0, st>>>(a);
        BT_LAUNCH("walk_fill");
    }
    BT_CUDA(cudaStreamSynchronize(st));
}

}  // namespace bt
