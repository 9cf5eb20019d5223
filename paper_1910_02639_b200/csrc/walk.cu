// walk.cu -- FindNeighbors (Alg. 2) for all particles on the device.
//
// Work unit = up to 64 queries of one leaf bucket (the paper's "blocked
// approach", Sec. IV-E: particles are in tree order, so a unit's queries
// are spatial neighbours).  One warp per unit; persistent warps pull units
// from an atomic counter.
//
// Test pass (count), per unit:
//   A10  breadth-first descent from the root with Eq. 5 index ranges of the
//        unit's query box widened by R'_u = max_i R'_i (lemma L1/L2,
//        DESIGN.md): all cells of all frontier nodes of a level are flattened
//        over the 32 lanes; empty cells skipped, internal cells form the next
//        frontier, leaf cells are culled by their tight box (L3) and queued;
//        queued leaves' particles are staged (flattened, two loads in flight
//        per lane), culled per particle against the query box in fp64 (L3),
//        as fp32 coordinates relative to the unit centre;
//   A11  lanes = candidates (two per lane, packed f32x2), loop over queries:
//        s32 < A_i -> certainly a neighbor, s32 >= B_i -> certainly not, else
//        the exact fp64 predicate ((dx*dx + dy*dy) + dz*dz) < (2h)^2 decides
//        (lemma L4).  __ballot_sync gives a 64-bit
//        neighbor mask per (64-candidate chunk, query), kept in shared memory;
//        __popc of the masks are the counts; masks and the chunk's candidate
//        indices are recorded in an arena for the fill pass.
// Scan (A12): offsets = exclusive scan of counts.
// Fill pass (A13): replay the recorded masks: __popc(mask & lanemask_lt) is
//        each neighbor's slot in its CSR row; coalesced row writes.
#include <algorithm>
#include <cfloat>

#include "common.cuh"
#include "scan.cuh"

namespace bt {

namespace {

constexpr int kQ = 64;          // queries per unit (== build.cu kUnitQ)
constexpr int kCand = 256;      // staged candidates per batch
constexpr int kChunks = kCand / 64;
constexpr int kLeafCap = 64;    // queued candidate leaves
constexpr int kWarpsPerBlock = 4;
constexpr int kWalkThreads = kWarpsPerBlock * 32;
constexpr int kFillThreads = 256;

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
    C_LOADED = 10,   // particle records loaded by staging (before the cull)
    C_N = 16
};

using Batch = WalkBatch;

struct WarpSmem {
    float4 q0[kQ];                         // ax, ax, ay, ay  (fp32, relative to the unit centre)
    float4 q1[kQ];                         // az, az, A, B    (certain-accept / certain-reject)
    int32_t qself[kQ];                     // batch slot of the query itself, -1 if not staged in this batch
    float2 px[kCand / 2], py[kCand / 2], pz[kCand / 2];  // chunk k, lane l: (c[64k+l], c[64k+32+l])
    int32_t cpos[kCand];                   // tree position of each staged candidate
    int32_t corig[kCand];                  // caller index of each staged candidate
    unsigned long long mask[kChunks][kQ];  // neighbor masks of the batch
    int32_t lbeg[kLeafCap + 1];              // queued leaves: first tree position
    int32_t lpre[kLeafCap + 1];            // queued leaves: exclusive prefix of counts
    float4 loff[kLeafCap + 1];             // queued leaves: fl32(c_leaf - c_unit), w = 1 if staged from rec32
};

struct WalkArgs {
    const double4 *rec;
    const float4 *rec32;
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
    int32_t *front;           // per-warp frontier scratch: 2 x front_cap node ids
    int64_t front_cap;
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
__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
    return ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
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

// Bound on |a - (x - c)| for the fp32 relative coordinates a of every query
// and staged candidate of a unit (lemma L4): queries use a = fl32(fl64(x - c))
// (error <= u E + w (1+u) E + 2^-149); candidates staged from the compact
// records use a = fl32(r32 + fl32(fl64(c_leaf - c))) with r32 =
// fl32(fl64(x - c_leaf)), only for leaves of half-extent H <= 0.999 E, whose
// error is <= (u + w(1+u))(H + D) + w(|x - c| + ...) + 3 2^-149 <= 4.0001 w E +
// 3 2^-149 (D = |c_leaf - c| <= H + E).  One bound covers both.
__device__ __forceinline__ double l4_eps(double E) { return 4.01 * 0x1p-24 * E + 0x1p-147; }

// Lemma L4: thresholds A <= B (fp32) such that for the
// fp32 squared distance s32 of a pair whose coordinates relative to the unit
// centre are bounded by E (per axis),
//   s32 <  A  =>  fp64 predicate true,     s32 >= B  =>  fp64 predicate false.
// All slack factors round the bounds outward.
__device__ __forceinline__ void l4_thresholds(double T, double E, double eps, bool exact_only, float &A, float &B) {
    const double u = 0x1p-53, w = 0x1p-24;
    if (exact_only || !(E < 1e15)) {
        A = 0.0f;
        B = __int_as_float(0x7f800000);  // +inf: every pair goes to the fp64 predicate
        return;
    }
    const double a0 = 2.0 * eps * (1.0 + w) + 0x1p-150;        // |d - D| <= a0 + w |D|
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

// squared distance from a point to the box [lo, hi], fp64 rounded ops
__device__ __forceinline__ double box_gap2(double x, double y, double z, double lx, double ly, double lz, double hx,
                                           double hy, double hz) {
    double gx = fmax(0.0, fmax(__dsub_rn(lx, x), __dsub_rn(x, hx)));
    double gy = fmax(0.0, fmax(__dsub_rn(ly, y), __dsub_rn(y, hy)));
    double gz = fmax(0.0, fmax(__dsub_rn(lz, z), __dsub_rn(z, hz)));
    return __dadd_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)), __dmul_rn(gz, gz));
}

// per-unit state, held in registers (every field warp-uniform unless noted)
struct Unit {
    int64_t id;
    int q0, nq;
    double lo[3], hi[3], c[3];
    double Ru, Ru2;
    float blo[3], bhi[3];   // query box in fp32 relative coordinates
    float cull2;            // fp32 Minkowski cull threshold (conservative)
    double E;               // a-priori bound |x - c| per axis (L4)
    int ncand;        // staged candidates in the current batch
    int nleaf;        // queued leaves
    int prev_batch;
    int cnt0, cnt1;   // per lane: counts of queries lane, lane + 32
    long long staged, loaded, tests, exact;
};

// s32 of candidate pair (lane, lane + 32) of chunk k against query q
struct Pair32 {
    float s0, s1;
};
__device__ __forceinline__ Pair32 s32_pair(unsigned long long cx, unsigned long long cy, unsigned long long cz,
                                           const float4 &Q0, const float4 &Q1) {
    const unsigned long long dx = f2_sub(cx, pk(Q0.x, Q0.y));
    const unsigned long long dy = f2_sub(cy, pk(Q0.z, Q0.w));
    const unsigned long long dz = f2_sub(cz, pk(Q1.x, Q1.y));
    unsigned long long s = f2_mul(dx, dx);
    s = f2_fma(dy, dy, s);
    s = f2_fma(dz, dz, s);
    return Pair32{__uint_as_float((unsigned)s), __uint_as_float((unsigned)(s >> 32))};
}

// The exact band of lemma L4 (rare): redo the batch's pairs, and let the fp64
// predicate itself decide every pair with A <= s32 < B.
__device__ __noinline__ void resolve_band(WarpSmem &S, Unit &U, int lane, const WalkArgs &a, int nch) {
    for (int k = 0; k < nch; k++) {
        const float2 vx = S.px[32 * k + lane], vy = S.py[32 * k + lane], vz = S.pz[32 * k + lane];
        const unsigned long long cx = pk(vx.x, vx.y), cy = pk(vy.x, vy.y), cz = pk(vz.x, vz.y);
        const int cp0 = S.cpos[64 * k + lane], cp1 = S.cpos[64 * k + 32 + lane];
        for (int q = 0; q < U.nq; q++) {
            const float4 Q0 = S.q0[q], Q1 = S.q1[q];
            const Pair32 p = s32_pair(cx, cy, cz, Q0, Q1);
            const bool u0 = !(p.s0 < Q1.z) && p.s0 < Q1.w, u1 = !(p.s1 < Q1.z) && p.s1 < Q1.w;
            if (!__any_sync(0xffffffffu, u0 || u1)) continue;
            const int qp = U.q0 + q;
            const double4 Qr = a.rec[qp];
            const double t = __dmul_rn(2.0, a.h_tree[qp]);
            const double T = __dmul_rn(t, t);
            bool e0 = false, e1 = false;
            if (u0) e0 = cp0 != qp && exact_pair(Qr.x, Qr.y, Qr.z, T, a.rec[cp0]);
            if (u1) e1 = cp1 != qp && exact_pair(Qr.x, Qr.y, Qr.z, T, a.rec[cp1]);
            const unsigned m0 = __ballot_sync(0xffffffffu, e0), m1 = __ballot_sync(0xffffffffu, e1);
            if (lane == 0) S.mask[k][q] |= ((unsigned long long)m1 << 32) | m0;
            U.exact += __popc(__ballot_sync(0xffffffffu, u0)) + __popc(__ballot_sync(0xffffffffu, u1));
            __syncwarp();
        }
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// A11: test the staged batch against all queries, record it, count.
// ---------------------------------------------------------------------------
__device__ __noinline__ void test_batch(WarpSmem &S, Unit &U, int lane, const WalkArgs &a) {
    const int ncand = U.ncand;
    const int nq = U.nq;
    const int nch = (ncand + 63) >> 6;
    const float inf = __int_as_float(0x7f800000);
    // pad the last chunk: +inf coordinates never pass (s32 = +inf)
    for (int c = ncand + lane; c < nch * 64; c += 32) {
        const int k = c >> 6, l = c & 31, hi = (c >> 5) & 1;
        reinterpret_cast<float *>(&S.px[32 * k + l])[hi] = inf;
        reinterpret_cast<float *>(&S.py[32 * k + l])[hi] = inf;
        reinterpret_cast<float *>(&S.pz[32 * k + l])[hi] = inf;
        S.corig[c] = -1;
        S.cpos[c] = -1;
    }
    __syncwarp();
    // Hot loop, branch free, register blocked: 4 queries held in registers,
    // candidate pairs of each chunk streamed from shared memory.  Certain
    // accepts (s32 < A) go into the masks; the ballots of s32 < B are compared
    // with them, and any difference (a pair in the band [A, B) of lemma L4) is
    // resolved afterwards by the fp64 predicate.  Queries are padded to a
    // multiple of 4 with A = B = 0.
    unsigned diff = 0;
    for (int q = 0; q < nq; q += 4) {
        unsigned long long qx[4], qy[4], qz[4];
        float A[4], B[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const float4 Q0 = S.q0[q + i], Q1 = S.q1[q + i];
            qx[i] = pk(Q0.x, Q0.y);
            qy[i] = pk(Q0.z, Q0.w);
            qz[i] = pk(Q1.x, Q1.y);
            A[i] = Q1.z;
            B[i] = Q1.w;
        }
        for (int k = 0; k < nch; k++) {
            const float2 vx = S.px[32 * k + lane], vy = S.py[32 * k + lane], vz = S.pz[32 * k + lane];
            const unsigned long long cx = pk(vx.x, vx.y), cy = pk(vy.x, vy.y), cz = pk(vz.x, vz.y);
            unsigned long long m[4];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const unsigned long long dx = f2_sub(cx, qx[i]);
                const unsigned long long dy = f2_sub(cy, qy[i]);
                const unsigned long long dz = f2_sub(cz, qz[i]);
                unsigned long long s = f2_mul(dx, dx);
                s = f2_fma(dy, dy, s);
                s = f2_fma(dz, dz, s);
                const float s0 = __uint_as_float((unsigned)s), s1 = __uint_as_float((unsigned)(s >> 32));
                const unsigned m0 = __ballot_sync(0xffffffffu, s0 < A[i]);
                const unsigned m1 = __ballot_sync(0xffffffffu, s1 < A[i]);
                const unsigned n0 = __ballot_sync(0xffffffffu, s0 < B[i]);
                const unsigned n1 = __ballot_sync(0xffffffffu, s1 < B[i]);
                diff |= (n0 ^ m0) | (n1 ^ m1);
                m[i] = ((unsigned long long)m1 << 32) | m0;
            }
            if (lane == 0) {
                ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(&S.mask[k][q]);
                dst[0] = make_ulonglong2(m[0], m[1]);
                dst[1] = make_ulonglong2(m[2], m[3]);
            }
        }
    }
    __syncwarp();
    if (diff) resolve_band(S, U, lane, a, nch);
    __syncwarp();
    // self is never its own neighbor (R12); counts; record the batch
    for (int q = lane; q < nq; q += 32) {
        const int sl = S.qself[q];
        if (sl >= 0) S.mask[sl >> 6][q] &= ~(1ull << (sl & 63));
        int c = 0;
        for (int k = 0; k < nch; k++) c += __popcll(S.mask[k][q]);
        if (q < 32) U.cnt0 += c;
        else U.cnt1 += c;
        S.qself[q] = -1;
    }
    long long mb = 0, cb = 0, bi = 0;
    if (lane == 0) {
        mb = atomicAdd((unsigned long long *)&a.ctr[C_MASK], (unsigned long long)(nch * nq));
        cb = atomicAdd((unsigned long long *)&a.ctr[C_CAND], (unsigned long long)(nch * 64));
        bi = atomicAdd((unsigned long long *)&a.ctr[C_BATCH], 1ull);
    }
    mb = __shfl_sync(0xffffffffu, mb, 0);
    cb = __shfl_sync(0xffffffffu, cb, 0);
    bi = __shfl_sync(0xffffffffu, bi, 0);
    const bool record = (mb + (long long)nch * nq <= a.mask_cap) && (cb + (long long)nch * 64 <= a.cand_cap) &&
                        (bi < a.batch_cap);
    __syncwarp();
    if (record) {
        for (int c = lane; c < nch * 64; c += 32) a.cands[cb + c] = S.corig[c];
        for (int w = lane; w < nch * nq; w += 32) a.masks[mb + w] = S.mask[w / nq][w % nq];
        if (lane == 0) {
            a.batches[bi] = Batch{mb, cb, ncand, -1};
            if (U.prev_batch >= 0) a.batches[U.prev_batch].next = (int)bi;
            else a.head[U.id] = (int)bi;
        }
        U.prev_batch = (int)bi;
    }
    U.tests += (long long)ncand * nq;
    U.ncand = 0;
    __syncwarp();
}

// ---------------------------------------------------------------------------
// Stage the queued leaves' particles (flattened over the lanes, two loads in
// flight per lane), per-particle cull (L3), fp32 relative coordinates.
// ---------------------------------------------------------------------------
__device__ __noinline__ void stage_leaves(WarpSmem &S, Unit &U, int lane, const WalkArgs &a) {
    const unsigned lt = lanemask_lt();
    const int nl = U.nleaf;
    // unit constants in registers (U lives in local memory across calls)
    const float blo0 = U.blo[0], blo1 = U.blo[1], blo2 = U.blo[2];
    const float bhi0 = U.bhi[0], bhi1 = U.bhi[1], bhi2 = U.bhi[2];
    const float cull2 = U.cull2;
    const double c0 = U.c[0], c1 = U.c[1], c2 = U.c[2];
    const int q0 = U.q0, nq = U.nq;
    int ncand = U.ncand;
    int staged = 0, loaded = 0;
    // exclusive prefix of the queued leaf counts (lpre was filled with counts)
    int carry = 0;
    for (int i0 = 0; i0 < nl; i0 += 32) {
        const int i = i0 + lane;
        const int v = (i < nl) ? S.lpre[i] : 0;
        int inc = v;
        for (int d = 1; d < 32; d <<= 1) {
            int o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += o;
        }
        if (i < nl) S.lpre[i] = carry + inc - v;
        carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) S.lpre[nl] = carry;
    __syncwarp();
    const int total = carry;
    int owner = 0;  // queued leaf that holds the next flattened position
    // gather one group of 64 flattened positions: record, leaf offset, position
    auto gather = [&](int p0, float4 (&r)[2], float4 (&of)[2], int (&pos)[2], bool (&valid)[2]) {
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int w0 = p0 + 32 * h;
            // owners of the 32 positions [w0, w0 + 32): leaf starts inside the window
            const int nxt = owner + 1 + lane;
            const int st = (nxt <= nl) ? S.lpre[nxt] : 0x7fffffff;
            const int off = st - w0;  // >= 1 for leaves after `owner` (until it crosses)
            const unsigned bits = __reduce_or_sync(0xffffffffu, (off >= 1 && off < 32) ? (1u << off) : 0u);
            const int mine = owner + __popc(bits & ((2u << lane) - 1u));
            const unsigned past = __ballot_sync(0xffffffffu, off <= 32);  // starts at or before w0 + 32
            const int p = w0 + lane;
            valid[h] = p < total;
            pos[h] = valid[h] ? S.lbeg[mine] + (p - S.lpre[mine]) : 0;
            of[h] = S.loff[mine];
            owner += __popc(past);
            r[h] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (valid[h]) {
                if (of[h].w != 0.0f) {
                    r[h] = a.rec32[pos[h]];
                } else {  // large leaf: exact fp64 record, a = fl32(fl64(x - c))
                    const double4 d = a.rec[pos[h]];
                    r[h] = make_float4(__double2float_rn(__dsub_rn(d.x, c0)), __double2float_rn(__dsub_rn(d.y, c1)),
                                       __double2float_rn(__dsub_rn(d.z, c2)),
                                       __int_as_float((int)__double_as_longlong(d.w)));
                    of[h].x = of[h].y = of[h].z = 0.0f;
                }
            }
        }
    };
    float4 r[2], of[2];
    int pos[2];
    bool valid[2];
    if (total > 0) gather(0, r, of, pos, valid);
    for (int p0 = 0; p0 < total; p0 += 64) {
        // prefetch the next group before culling this one (loads in flight)
        float4 rn[2], ofn[2];
        int posn[2];
        bool validn[2] = {false, false};
        if (p0 + 64 < total) gather(p0 + 64, rn, ofn, posn, validn);
        if (ncand + 64 > kCand) {
            U.ncand = ncand;
            test_batch(S, U, lane, a);
            ncand = 0;
        }
#pragma unroll
        for (int h = 0; h < 2; h++) {
            // fp32 relative coordinates (compact: fl32(r32 + fl32(c_leaf - c)); the
            // fp64 path already holds fl32(fl64(x - c)) with a zero offset) and the
            // conservative fp32 Minkowski cull against the query box (L3 / L4)
            const float ax = __fadd_rn(r[h].x, of[h].x);
            const float ay = __fadd_rn(r[h].y, of[h].y);
            const float az = __fadd_rn(r[h].z, of[h].z);
            const float gx = fmaxf(0.0f, fmaxf(__fsub_rn(blo0, ax), __fsub_rn(ax, bhi0)));
            const float gy = fmaxf(0.0f, fmaxf(__fsub_rn(blo1, ay), __fsub_rn(ay, bhi1)));
            const float gz = fmaxf(0.0f, fmaxf(__fsub_rn(blo2, az), __fsub_rn(az, bhi2)));
            const float g2 = __fmaf_rn(gz, gz, __fmaf_rn(gy, gy, __fmul_rn(gx, gx)));
            const bool keep = valid[h] && g2 < cull2;
            const unsigned km = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const int slot = ncand + __popc(km & lt);
                const int ck = slot >> 6, cl = slot & 31, ch = (slot >> 5) & 1;
                reinterpret_cast<float *>(&S.px[32 * ck + cl])[ch] = ax;
                reinterpret_cast<float *>(&S.py[32 * ck + cl])[ch] = ay;
                reinterpret_cast<float *>(&S.pz[32 * ck + cl])[ch] = az;
                S.cpos[slot] = pos[h];
                S.corig[slot] = __float_as_int(r[h].w);
                const int qi = pos[h] - q0;
                if (qi >= 0 && qi < nq) S.qself[qi] = slot;
            }
            ncand += __popc(km);
            staged += __popc(km);
            loaded += __popc(__ballot_sync(0xffffffffu, valid[h]));
        }
#pragma unroll
        for (int h = 0; h < 2; h++) {
            r[h] = rn[h];
            of[h] = ofn[h];
            pos[h] = posn[h];
            valid[h] = validn[h];
        }
        __syncwarp();
    }
    U.ncand = ncand;
    U.staged += staged;
    U.loaded += loaded;
    U.nleaf = 0;
    __syncwarp();
}

// queue a leaf (if its tight box is within R'_u of the query box: L3)
__device__ __forceinline__ void queue_leaves(WarpSmem &S, Unit &U, int lane, const WalkArgs &a, bool is_leaf,
                                             int32_t leaf) {
    const unsigned lt = lanemask_lt();
    bool keep = false;
    float4 off = make_float4(0.f, 0.f, 0.f, 0.f);
    if (is_leaf) {
        const double2 *lb = reinterpret_cast<const double2 *>(a.leaf_box + 6 * (int64_t)leaf);
        const double2 b0 = lb[0], b1 = lb[1], b2 = lb[2];  // lo x,y | lo z, hi x | hi y,z
        double gx = fmax(0.0, fmax(__dsub_rn(b0.x, U.hi[0]), __dsub_rn(U.lo[0], b1.y)));
        double gy = fmax(0.0, fmax(__dsub_rn(b0.y, U.hi[1]), __dsub_rn(U.lo[1], b2.x)));
        double gz = fmax(0.0, fmax(__dsub_rn(b1.x, U.hi[2]), __dsub_rn(U.lo[2], b2.y)));
        double g2 = __dadd_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)), __dmul_rn(gz, gz));
        keep = g2 < U.Ru2;
        // leaf centre (as build.cu computed it) relative to the unit centre; the
        // compact records are usable when the leaf half-extent H <= 0.999 E (l4_eps)
        const double cx = 0.5 * (b0.x + b1.y), cy = 0.5 * (b0.y + b2.x), cz = 0.5 * (b1.x + b2.y);
        const double H = 0.5 * fmax(fmax(b1.y - b0.x, b2.x - b0.y), b2.y - b1.x);
        off = make_float4(__double2float_rn(__dsub_rn(cx, U.c[0])), __double2float_rn(__dsub_rn(cy, U.c[1])),
                          __double2float_rn(__dsub_rn(cz, U.c[2])), (H <= 0.999 * U.E) ? 1.0f : 0.0f);
    }
    const unsigned km = __ballot_sync(0xffffffffu, keep);
    if (!km) return;
    if (U.nleaf + __popc(km) > kLeafCap) stage_leaves(S, U, lane, a);
    if (keep) {
        const int slot = U.nleaf + __popc(km & lt);
        S.lbeg[slot] = a.leaf_begin[leaf];
        S.lpre[slot] = a.leaf_count[leaf];  // counts; stage_leaves turns them into a prefix
        S.loff[slot] = off;
    }
    U.nleaf += __popc(km);
    __syncwarp();
}

#ifndef BT_WALK_MIN_BLOCKS
#define BT_WALK_MIN_BLOCKS 5
#endif
__global__ void __launch_bounds__(kWalkThreads, BT_WALK_MIN_BLOCKS) test_kernel(WalkArgs a) {
    __shared__ WarpSmem smem[kWarpsPerBlock];
    const int lane = threadIdx.x & 31;
    WarpSmem &S = smem[threadIdx.x >> 5];
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int32_t *const front_base = a.front + gwarp * 2 * a.front_cap;
    const unsigned lt = lanemask_lt();
    long long staged = 0, loaded = 0, tests = 0, exact = 0;

    for (;;) {
        unsigned long long uid = 0;
        if (lane == 0) uid = atomicAdd((unsigned long long *)&a.ctr[C_WORK], 1ull);
        uid = __shfl_sync(0xffffffffu, uid, 0);
        if (uid >= (unsigned long long)a.n_units) break;
        const int4 UU = a.units[uid];
        Unit U;
        U.id = (int64_t)uid;
        U.q0 = UU.y;
        U.nq = UU.z;
        U.ncand = U.nleaf = 0;
        U.prev_batch = -1;
        U.cnt0 = U.cnt1 = 0;
        U.staged = U.loaded = U.tests = U.exact = 0;
        if (lane == 0) a.head[uid] = -1;

        // ---- queries: coordinates, (2h)^2, R', box
        double qx[2], qy[2], qz[2], qT[2];
        int32_t qo[2] = {0, 0};
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        double Ru = 0.0;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int k = lane + 32 * h;
            qx[h] = qy[h] = qz[h] = qT[h] = 0.0;
            if (k < U.nq) {
                const double4 r = a.rec[U.q0 + k];
                const double t = __dmul_rn(2.0, a.h_tree[U.q0 + k]);  // 2h (exact)
                qx[h] = r.x;
                qy[h] = r.y;
                qz[h] = r.z;
                qT[h] = __dmul_rn(t, t);
                qo[h] = (int32_t)__double_as_longlong(r.w);
                // R' = 2h (1 + 2^-40) + 2^-50 M   (lemma L1/L2)
                Ru = fmax(Ru, __dadd_rn(__dmul_rn(t, 1.0 + 0x1p-40), __dmul_rn(0x1p-50, a.M)));
                lo[0] = fmin(lo[0], r.x); lo[1] = fmin(lo[1], r.y); lo[2] = fmin(lo[2], r.z);
                hi[0] = fmax(hi[0], r.x); hi[1] = fmax(hi[1], r.y); hi[2] = fmax(hi[2], r.z);
            }
            S.qself[k] = -1;
        }
        double E = 0.0, Mu = 0.0;
        // a unit holding its whole leaf has the leaf's tight box as its query box
        const bool whole = U.nq == a.leaf_count[UU.x];
        const double *lb = a.leaf_box + 6 * (int64_t)UU.x;
        for (int l = 0; l < 3; l++) {
            U.lo[l] = whole ? lb[l] : warp_min(lo[l]);
            U.hi[l] = whole ? lb[3 + l] : warp_max(hi[l]);
            U.c[l] = 0.5 * (U.lo[l] + U.hi[l]);
            E = fmax(E, 0.5 * (U.hi[l] - U.lo[l]));
            Mu = fmax(Mu, fmax(fabs(U.lo[l]), fabs(U.hi[l])));
        }
        U.Ru = warp_max(Ru);
        U.Ru2 = __dmul_rn(U.Ru, U.Ru);
        // a-priori bound |x - c| <= E per axis for queries and staged candidates (L4)
        E = (E + U.Ru) * 1.0001 + 4.0 * 0x1p-53 * Mu;
        U.E = E;
        {
            // fp32 images of the query box and the conservative cull radius
            // (R'_u + 4 eps)(1 + 2^-20), eps = the fp32 coordinate error bound of L4
            const double eps = l4_eps(E);
            for (int l = 0; l < 3; l++) {
                U.blo[l] = __double2float_rn(__dsub_rn(U.lo[l], U.c[l]));
                U.bhi[l] = __double2float_rn(__dsub_rn(U.hi[l], U.c[l]));
            }
            const double rc = (U.Ru + 4.0 * eps) * (1.0 + 0x1p-20);
            const double rc2 = rc * rc * (1.0 + 0x1p-40);
            U.cull2 = (rc2 < 3.0e38) ? __double2float_ru(rc2) : __int_as_float(0x7f800000);
        }
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int k = lane + 32 * h;
            if (k < U.nq) {
                const float ax = __double2float_rn(__dsub_rn(qx[h], U.c[0]));
                const float ay = __double2float_rn(__dsub_rn(qy[h], U.c[1]));
                const float az = __double2float_rn(__dsub_rn(qz[h], U.c[2]));
                float A, B;
                l4_thresholds(qT[h], E, l4_eps(E), a.exact_only != 0, A, B);
                S.q0[k] = make_float4(ax, ax, ay, ay);
                S.q1[k] = make_float4(az, az, A, B);
            } else {
                S.q0[k] = make_float4(0.f, 0.f, 0.f, 0.f);
                S.q1[k] = make_float4(0.f, 0.f, 0.f, 0.f);  // A = B = 0: never a neighbor
            }
        }
        __syncwarp();

        // ---- A10: breadth-first descent, all cells of a level flattened over the lanes
        if (a.root_is_leaf) {
            queue_leaves(S, U, lane, a, lane == 0, 0);
        } else {
            int32_t *fcur = front_base, *fnext = front_base + a.front_cap;
            int nf = 1;
            if (lane == 0) fcur[0] = 0;
            __syncwarp();
            while (nf > 0) {
                int nnext = 0;
                for (int f0 = 0; f0 < nf; f0 += 32) {
                    const int fi = f0 + lane;
                    int b = 0, r0x = 0, r0y = 0, r0z = 0, nx = 1, ny = 1;
                    long long cb = 0, tot = 0;
                    if (fi < nf) {
                        const NodeRec &nd = a.nodes[fcur[fi]];
                        b = nd.b;
                        cb = nd.cell_base;
                        int r0[3], r1[3];
                        for (int l = 0; l < 3; l++) {
                            r0[l] = cell_coord(__dsub_rn(U.lo[l], U.Ru), nd.lo[l], nd.ext[l], b);
                            r1[l] = cell_coord(__dadd_rn(U.hi[l], U.Ru), nd.lo[l], nd.ext[l], b);
                        }
                        r0x = r0[0];
                        r0y = r0[1];
                        r0z = r0[2];
                        nx = r1[0] - r0[0] + 1;
                        ny = r1[1] - r0[1] + 1;
                        tot = (long long)nx * ny * (r1[2] - r0[2] + 1);
                    }
                    // inclusive scan of the cell counts over the lanes
                    long long inc = tot;
                    for (int d = 1; d < 32; d <<= 1) {
                        long long o = __shfl_up_sync(0xffffffffu, inc, d);
                        if (lane >= d) inc += o;
                    }
                    const long long start = inc - tot;
                    const long long T = __shfl_sync(0xffffffffu, inc, 31);
                    int owner = 0;
                    for (long long c0 = 0; c0 < T; c0 += 32) {
                        // owner lane of cell g = c0 + lane (node starts inside the window)
                        const long long off = start - c0;
                        const unsigned bits =
                            __reduce_or_sync(0xffffffffu, (lane > owner && off >= 1 && off < 32) ? (1u << off) : 0u);
                        const int o = owner + __popc(bits & ((2u << lane) - 1u));
                        const unsigned past = __ballot_sync(0xffffffffu, lane > owner && off <= 32);
                        const int ob = __shfl_sync(0xffffffffu, b, o);
                        const long long ocb = __shfl_sync(0xffffffffu, cb, o);
                        const int ox = __shfl_sync(0xffffffffu, r0x, o), oy = __shfl_sync(0xffffffffu, r0y, o),
                                  oz = __shfl_sync(0xffffffffu, r0z, o);
                        const int onx = __shfl_sync(0xffffffffu, nx, o), ony = __shfl_sync(0xffffffffu, ny, o);
                        const long long ostart = __shfl_sync(0xffffffffu, start, o);
                        owner += __popc(past);
                        const long long g = c0 + lane;
                        bool is_leaf = false, is_node = false;
                        int32_t code = -1;
                        if (g < T) {
                            const int local = (int)(g - ostart);
                            const int cx = ox + local % onx;
                            const int cy = oy + (local / onx) % ony;
                            const int cz = oz + local / (onx * ony);
                            const long long j = cx + (long long)cy * ob + (long long)cz * ob * ob;  // Eq. 3
                            code = a.cells[ocb + j];
                            is_leaf = code >= 0;
                            is_node = code <= -2;
                        }
                        const unsigned nm = __ballot_sync(0xffffffffu, is_node);
                        if (is_node) fnext[nnext + __popc(nm & lt)] = code_node(code);
                        nnext += __popc(nm);
                        queue_leaves(S, U, lane, a, is_leaf, code);
                    }
                }
                __syncwarp();
                int32_t *tmp = fcur;
                fcur = fnext;
                fnext = tmp;
                nf = nnext;
            }
        }
        if (U.nleaf > 0) stage_leaves(S, U, lane, a);
        if (U.ncand > 0 || U.prev_batch < 0) test_batch(S, U, lane, a);
        if (lane < U.nq) a.counts[qo[0]] = U.cnt0;
        if (lane + 32 < U.nq) a.counts[qo[1]] = U.cnt1;
        staged += U.staged;
        loaded += U.loaded;
        tests += U.tests;
        exact += U.exact;
        __syncwarp();
    }
    if (lane == 0) {
        atomicAdd((unsigned long long *)&a.ctr[C_STAGED], (unsigned long long)staged);
        atomicAdd((unsigned long long *)&a.ctr[C_LOADED], (unsigned long long)loaded);
        atomicAdd((unsigned long long *)&a.ctr[C_TESTS], (unsigned long long)tests);
        atomicAdd((unsigned long long *)&a.ctr[C_EXACT], (unsigned long long)exact);
    }
}

// ---------------------------------------------------------------------------
// Fill pass: replay the recorded masks into the CSR rows.  Per unit and batch
// the candidate indices and masks are staged in shared memory; for each
// (chunk, query) mask word, lane l owns candidates 64k + l and 64k + 32 + l,
// and __popc(mask & lanemask_lt) gives its slot in the query's row (row order
// unspecified, R15).  The next write position of each query lives in shared
// memory.
// ---------------------------------------------------------------------------
constexpr int kFillWarps = kFillThreads / 32;

struct FillSmem {
    unsigned long long wr[kQ];                 // next write position of each query's row
    unsigned long long mask[kChunks * kQ];     // the batch's masks, [k][q]
    int32_t cand[kCand];                       // the batch's candidate caller indices
};

__global__ void __launch_bounds__(kFillThreads) fill_kernel(WalkArgs a) {
    __shared__ FillSmem fsm[kFillWarps];
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
    FillSmem &F = fsm[threadIdx.x >> 5];
    for (;;) {
        unsigned long long u = 0;
        if (lane == 0) u = atomicAdd((unsigned long long *)&a.ctr[C_WORK2], 1ull);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= (unsigned long long)a.n_units) break;
        const int4 U = a.units[u];
        const int nq = U.z;
        for (int q = lane; q < nq; q += 32)
            F.wr[q] = (unsigned long long)a.offsets[(int32_t)__double_as_longlong(a.rec[U.y + q].w)];
        for (int b = a.head[u]; b >= 0;) {
            const Batch B = a.batches[b];
            const int nch = (B.ncand + 63) >> 6;
            __syncwarp();
            for (int c = lane; c < nch * 64; c += 32) F.cand[c] = a.cands[B.cand_base + c];
            for (int w = lane; w < nch * nq; w += 32) F.mask[w] = a.masks[B.mask_base + w];
            __syncwarp();
            for (int k = 0; k < nch; k++) {
                const int32_t c0 = F.cand[64 * k + lane], c1 = F.cand[64 * k + 32 + lane];
                const unsigned long long *mk = F.mask + k * nq;
                for (int q = 0; q < nq; q++) {
                    const unsigned long long m = mk[q];
                    if (m == 0ull) continue;
                    const unsigned long long base = F.wr[q];
                    const unsigned lo = (unsigned)m, hi = (unsigned)(m >> 32);
                    const int plo = __popc(lo);
                    if ((lo >> lane) & 1u) a.nbr[base + __popc(lo & lt)] = c0;
                    if ((hi >> lane) & 1u) a.nbr[base + plo + __popc(hi & lt)] = c1;
                    if (lane == 0) F.wr[q] = base + plo + __popc(hi);
                }
                __syncwarp();
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

    // persistent grids: all resident warps
    int per_sm = 0, per_sm_fill = 0;
    BT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, test_kernel, kWalkThreads, 0));
    BT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_fill, fill_kernel, kFillThreads, 0));
    per_sm = std::max(per_sm, 1);
    per_sm_fill = std::max(per_sm_fill, 1);
    const unsigned grid = (unsigned)(sms * per_sm);
    const unsigned grid_fill = (unsigned)(sms * per_sm_fill);
    const int64_t nwarps = (int64_t)grid * kWarpsPerBlock;
    // frontier scratch: a unit's frontier holds each internal node at most once
    const int64_t front_cap = std::max<int64_t>(t.n_nodes, 1);
    t.front.reserve(nwarps * 2 * front_cap, 0);
    t.head.reserve(t.n_units, 0);

    // the recorded masks of a previous test pass are reused by a fill-only
    // call when the tree, h pointer, exactness mode and h checksum all match
    const bool have_record = t.rec_valid && t.rec_h == h && t.rec_hsum == hsum && t.rec_exact == g_exact_only;
    const bool run_test = count_pass || !have_record;

    WalkArgs a{};
    a.rec = t.rec.p;
    a.rec32 = t.rec32.p;
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
    a.front = t.front.p;
    a.front_cap = front_cap;
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
        static thread_local double mask_per_q = 12.0, cand_per_q = 24.0, batch_per_unit = 3.0;
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
            BT_CUDA(cudaMemsetAsync(t.counters.p + C_HSUM + 1, 0, (C_N - C_HSUM - 1) * sizeof(int64_t), st));
            {
                Phase ph("search.count");
                test_kernel<<<grid, kWalkThreads, 0, st>>>(a);
                BT_LAUNCH("walk_test");
            }
            long long hc[C_N];
            BT_CUDA(cudaMemcpyAsync(hc, t.counters.p, C_N * sizeof(long long), cudaMemcpyDeviceToHost, st));
            BT_CUDA(cudaStreamSynchronize(st));
            t.staged = hc[C_STAGED];
            t.loaded = hc[C_LOADED];
            t.tests = hc[C_TESTS];
            t.exact_tests = hc[C_EXACT];
            const bool fits = hc[C_MASK] <= a.mask_cap && hc[C_CAND] <= a.cand_cap && hc[C_BATCH] <= a.batch_cap;
            mask_per_q = std::max(mask_per_q, 1.1 * (double)hc[C_MASK] / (double)n);
            cand_per_q = std::max(cand_per_q, 1.1 * (double)hc[C_CAND] / (double)n);
            batch_per_unit =
                std::max(batch_per_unit, 1.1 * (double)hc[C_BATCH] / (double)std::max<int64_t>(1, t.n_units));
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
        fill_kernel<<<grid_fill, kFillThreads, 0, st>>>(a);
        BT_LAUNCH("walk_fill");
    }
    BT_CUDA(cudaStreamSynchronize(st));
}

}  // namespace bt
