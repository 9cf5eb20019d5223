// walk.cu -- FindNeighbors (Alg. 2) for all particles on the device.
//
// Work unit = up to 64 queries of one leaf bucket (the paper's "blocked
// approach", Sec. IV-E: particles are in tree order, so a unit's queries
// are spatial neighbours).  One warp per unit; persistent warps pull units
// (in Morton order of their leaf, build.cu) from an atomic counter.
//
// desc_kernel (A10): per unit, breadth-first descent from the root with Eq. 5
//   index ranges of the unit's query box widened by R'_u = max_i R'_i (lemma
//   L1/L2): all cells of all frontier nodes of a level are
//   flattened over the 32 lanes; empty cells skipped, internal cells form the
//   next frontier, leaf cells whose tight box is within R'_u of the query box
//   (L3) are appended to the unit's candidate-leaf list.
// walk_kernel (A10 staging + A11): per unit, the listed leaves' particles are
//   loaded (flattened over the lanes), culled per particle against the query
//   box (L3) and staged in shared memory as fp32 coordinates relative to the
//   unit centre, in blocks of 128.  Each block is tested against the unit's
//   queries: lanes = 4 candidates (two packed f32x2 pairs), loop over
//   queries; d = fl32(s32 - Mid_i) decides the certain cases (lemma L4),
//   pairs with |d| <= HW_i are decided by the exact fp64 predicate
//   ((dx*dx + dy*dy) + dz*dz) < (2h)^2.  __ballot_sync gives a 64-bit
//   neighbor mask per (64-candidate chunk, query); __popc of the masks are
//   the counts; masks and candidate caller indices are recorded per unit.
// Scan (A12): offsets = exclusive scan of counts.
// fill_kernel (A13): replay the recorded masks: __popc(mask & lanemask_lt) is
//   each neighbor's slot in its CSR row.
#include <algorithm>
#include <cfloat>
#include <type_traits>

#include "common.cuh"
#include "scan.cuh"

namespace bt {

namespace {

constexpr int kQ = 64;           // queries per unit (== build.cu kUnitQ)
constexpr int kBlk = 128;        // staged candidates per test block
constexpr int kStg = kBlk + 32;  // staged candidates per warp (shared memory): a block plus one window
constexpr int kGroup = 32;       // candidate leaves per staging group (one per lane)
constexpr int kGroupPos = 2048;  // positions a multi-leaf group may span (its leaf-start bitmap)
constexpr int kFrontCap = 512;   // shared-memory descent frontier per level
constexpr int kDescThreads = 128;
constexpr int kWalkThreads = 128;
#ifndef BT_FILL_THREADS
#define BT_FILL_THREADS 256
#endif
constexpr int kFillThreads = BT_FILL_THREADS;
#ifndef BT_FILL_CHUNKS
#define BT_FILL_CHUNKS 6
#endif
constexpr int kFillChunks = BT_FILL_CHUNKS;   // 64-candidate chunks per fill round (cfg 5 fill, with the prefix packs: 4 chunks 11.45 ms, 5 11.84, 6 10.66, 8 11.04)
constexpr long long kListSlab = 8192;     // leaf-list entries per warp allocation
constexpr long long kListReserve = 2048;  // more candidate leaves -> big-unit pass
constexpr long long kCandSlab = 16384;    // candidate slots per warp allocation
constexpr long long kMaskSlab = 8192;     // mask words per warp allocation

// device counters (int64 slots of TreeDev::counters)
enum {
    C_WORK = 0,      // unit counter (descent)
    C_MASK = 1,      // mask words allocated
    C_CAND = 2,      // candidate slots allocated
    C_LIST = 3,      // leaf-list entries allocated
    C_STAGED = 4,
    C_TESTS = 5,
    C_EXACT = 6,
    C_MAXC = 7,
    C_WORK2 = 8,     // unit counter (fill)
    C_HSUM = 9,      // checksum of h (bit patterns)
    C_LOADED = 10,   // particle records loaded by the staging (before the cull)
    C_WORK3 = 11,    // unit counter (walk)
    C_BIG = 12,      // units whose descent overflowed the shared-memory limits
    C_WORK4 = 13,    // unit counter (big-unit descent)
    C_NEEDC = 14,    // sum over units of `loaded` (bound on candidate slots)
    C_NEEDM = 15,    // sum over units of ceil(loaded / 64) * nq (bound on mask words)
    C_WORK5 = 16,    // unit counter (symmetric-criterion pass)
    C_OVER = 17,     // rows with more neighbors than the call's ngmax
    C_CSUM = 18,     // checksum of the test pass's counts: sum of counts[i] (2i + 1) mod 2^64
    C_OSUM = 19,     // the same checksum of a fill-only call's offsets differences
    C_OBAD = 20,     // a fill-only call's offsets are not a valid scan of the counts
    C_NZW = 21,      // recorded mask words with at least one neighbor
    C_HBAD = 22,     // the descent's fused gather met an h outside (0, 1e150]
    C_N = 23
};

struct WalkArgs {
    const double4 *rec;
    const float4 *rec32;
    const int32_t *perm;      // caller index of each tree position
    const double *h_tree;
    const double *h_src;      // non-null: the descent gathers h (caller order) into h_out itself
    double *h_out;            // (= h_tree)
    const NodeRec *nodes;
    const int32_t *cells;
    const int32_t *leaf_begin;
    const int32_t *leaf_count;
    const double *leaf_box;
    const LeafRec *leaf_rec;
    const int4 *units;
    int64_t n_units;
    double M;
    int root_is_leaf;
    int exact_only;
    int tree_order;           // bt_set_tree_order: per-particle arrays and neighbor indices in tree positions
    int32_t *front;           // big-unit pass: per-warp frontier scratch, 2 x front_cap node ids
    int64_t front_cap;
    UnitRun *urun;
    UnitPrep *uprep;          // gather count pass: the descent prepares each unit's walk geometry and
    float4 *qrec;             //   query records (tree positions), the walk loads them
    int32_t *ulist;
    long long list_cap;
    int32_t *counts;
    const int64_t *offsets;
    int32_t *nbr;
    long long *ctr;
    int32_t *cands;           // caller index of each candidate slot
    long long cand_cap;
    int64_t n_rec;            // particles (tree positions) -- bounds checks
    int64_t n_cells, n_leaves;  // cell-table entries, leaves -- bounds checks
    int64_t nbr_cap;          // int32 slots of nbr -- bounds checks
    unsigned long long *masks;
    long long mask_cap;
    int desc_batch;           // units claimed per atomic by the descent warps
    const double *m_tree;     // density mode: masses in tree order
    double *rho;              // density mode: output, caller order
    const double *leaf_hmax;  // symmetric mode: max h per leaf
    const double *node_hmax;  // symmetric mode: max h per internal node subtree
};

__device__ __forceinline__ double warp_min(double v) {
    for (int d = 16; d; d >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, d));
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
    for (int d = 16; d; d >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, d));
    return v;
}

// packed fp32 pair arithmetic (sm_100a FADD2 / FMUL2 / FFMA2): lo = first, hi = second
__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float lo_f(unsigned long long v) { return __uint_as_float((unsigned)v); }
__device__ __forceinline__ float hi_f(unsigned long long v) { return __uint_as_float((unsigned)(v >> 32)); }
__device__ __forceinline__ unsigned long long f2_add(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ int2 lds2iv(const int *p) {
    int2 v;
    asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"((unsigned)__cvta_generic_to_shared(p)));
    return v;
}

// Exact predicate (the definition): ((dx*dx + dy*dy) + dz*dz) < T, fp64, no FMA.
__device__ __forceinline__ bool exact_pair(double qx, double qy, double qz, double T, const double4 &c) {
    double dx = __dsub_rn(qx, c.x), dy = __dsub_rn(qy, c.y), dz = __dsub_rn(qz, c.z);
    double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    return d2 < T;
}

// Bound on |a - (x - c)| for the fp32 relative coordinates a of every query
// and candidate of a unit (lemma L4): queries use a = fl32(fl64(x - c))
// (error <= u E + w (1+u) E + 2^-149); candidates from the compact records
// use a = fl32(r32 + fl32(fl64(c_leaf - c))) with r32 = fl32(fl64(x - c_leaf)),
// only for leaves of half-extent H <= 7 E, whose error is
// <= (u + w(1+u))(H + D) + w(|x - c| + ...) + 3 2^-149 <= 16.01 w E + 3 2^-149
// (D = |c_leaf - c| <= H + E, so H + D <= 15 E).  One bound covers both.
__device__ __forceinline__ double l4_eps(double E) { return 16.02 * 0x1p-24 * E + 0x1p-146; }

// Lemma L4, expanded form.  The hot loop evaluates, per
// (candidate c, query q) with fp32 unit-relative coordinates,
//   v = fl(cx Qx + fl(cy Qy + fl(cz Qz + fl(Ac + Bq))))      (3 FMA + 1 add)
// with Ac = k fl(|c|^2) (per candidate), Q = -2 k q and Bq = fl32(k (|q|^2 -
// Mid)) (per query), k a power of two (exact scalings).  In exact arithmetic
// v = k (|c - q|^2 - Mid).  With E' >= every |coordinate| (E' = E(1 + 1e-6) +
// 5 eps: queries and kept candidates lie within E + 4 eps of the unit centre)
// the fp32 arithmetic errs by at most k G, G = u (60.1 E'^2 + 5.01 Mid_max)
// (u = 2^-24: |c|^2 in three roundings <= 9.01 u E'^2, Bq <= u (3E'^2 + Mid),
// four roundings of partial sums bounded by k (12 E'^2 + Mid)), and the inputs'
// representation error (<= eps per coordinate, so <= 2 eps per axis of c - q)
// moves |c - q|^2 from the exact S by <= 4 sqrt(3) eps sqrt(S) + 12 eps^2.
// So Err(S) = 4 sqrt3 eps sqrt(S) + 12 eps^2 + G bounds |v/k + Mid - S|; with
// T- = T (1 - 8 u64), T+ = T (1 + 8 u64) (the fp64 predicate's rounding) and
// S - Err(S) increasing on [T-, inf):
//   A = T- - Err(T-),  B = T+ + Err(T+),  HW >= max(|Mid - A|, |B - Mid|),
//   k = largest power of two <= 1/HW  =>  [t_acc, t_rej) = k [A - Mid, B - Mid)
//   lies inside [-1, 1], so |v| > 1 is certain: v < -1 => S < T- => neighbor,
//   v > 1 => S >= T+ => not; the band |v| <= 1 goes to the fp64 predicate.
// k = 0 ("force": exact-only, E >= 1e15, or a bound that fails) sends every
// pair to the fp64 predicate.  A unit uses the minimum k over its queries
// (1/k only grows, the band only widens).
// (t = 2h exactly, T = fl(t t): sqrt(T-) < t and sqrt(T+) <= t (1 + 2^-48)
// stand in for the square roots, and the power of two comes from hw's
// exponent -- no fp64 sqrt or division per query.)
__device__ __forceinline__ void l4_band(double T, double t, double E, double eps, bool exact_only, float &k,
                                        float &Mid) {
    k = 0.0f;
    Mid = 0.0f;
    if (exact_only || !(E < 1e15)) return;
    const double u = 0x1p-24, u64 = 0x1p-53, s3 = 1.7320508075688775;
    const double Ep = E * (1.0 + 1e-6) + 5.0 * eps;
    const double Tm = T * (1.0 - 8.0 * u64), Tp = T * (1.0 + 8.0 * u64);
    const double G = u * (60.1 * Ep * Ep + 5.01 * (2.0 * Tp));  // Mid <= B <= 2 T+ (checked below)
    // S - Err(S) increasing on [T-, inf): 2 sqrt3 eps <= sqrt(T-) / 2, sqrt(T-) >= t (1 - 2^-48)
    if (!(2.0 * s3 * eps * 1.0001 <= 0.5 * t * (1.0 - 0x1p-48))) return;
    const double A = Tm - (4.0 * s3 * eps * t + 12.0 * eps * eps + G) * 1.0001;                       // sqrt(T-) < t
    const double B = Tp + (4.0 * s3 * eps * t * (1.0 + 0x1p-48) + 12.0 * eps * eps + G) * 1.0001;  // sqrt(T+) bound
    if (!(A > 0.0) || !(B <= 2.0 * Tp)) return;
    const float M = __double2float_rn(0.5 * (A + B));
    double hw = fmax(fmax((double)M - A, B - (double)M), (double)M * 0x1p-23) * (1.0 + 0x1p-40);
    int e;
    const double f = frexp(hw, &e);                      // hw = f 2^e, f in [0.5, 1): 1/hw in (2^-e, 2^(1-e)]
    const double kd = ldexp(1.0, f == 0.5 ? 1 - e : -e); // largest power of two <= 1/hw
    // the expanded form's magnitudes stay far below fp32 overflow
    if (!(kd * (12.0 * Ep * Ep + (double)M) < 1e36) || !(2.0 * kd * Ep < 1e36)) return;
    k = (float)kd;
    Mid = M;
}

// Lemma L4 for the symmetric criterion (L4s): the hot
// loop evaluates u = fl(cx Qx + fl(cy Qy + fl(cz Qz + fl(Ac + B''q)))) with
// B''q = fl32(k |q|^2) (no Mid), then v_i = fl(u - k Mid_i) (query threshold)
// and v_j = fl(u - k Mid_j) (candidate threshold), Mid = fl32(T).  u errs by
// at most k G'', G'' = w 60.1 E'^2 (as G without the Mid terms); the final
// subtraction adds at most w |u - k Mid|, which moves the +-1 decision
// thresholds by < 2w.  So for every T <= Tmax of the unit,
//   HW(T) = w T + 8 u64 T + Err(T+) + G'' <= HW(Tmax)   (increasing in T)
// with Err(S) = 4 sqrt3 eps sqrt(S) + 12 eps^2 and sqrt(Tmax+) <= rmax (Tmax
// <= rmax^2: every threshold of the unit comes from an h whose R' <= rmax),
// and k = the largest power of two <= (1 - 2^-22) / HW(Tmax) makes v < -1 a
// certain neighbor, v > 1 a certain non-neighbor, |v| <= 1 the fp64 band.
// S - Err(S) must increase on [T-, inf) for the smallest threshold that can
// decide a pair: the smallest query threshold Tqmin (a candidate threshold
// Tj <= Tqmin is redundant, d2 < Tj implying d2 < Ti: such candidates carry
// +inf, never deciding).  k = 0: force (every pair to the fp64 predicate).
__device__ __forceinline__ float l4_band_sym(double Tqmin, double rmax, double E, double eps, bool exact_only) {
    if (exact_only || !(E < 1e15) || !(rmax < 1e15)) return 0.0f;
    const double u = 0x1p-24, u64 = 0x1p-53, s3 = 1.7320508075688775;
    const double Ep = E * (1.0 + 1e-6) + 5.0 * eps;
    const double Tmax = rmax * rmax * (1.0 + 0x1p-40);
    if (!(2.0 * s3 * eps * 1.0001 <= 0.5 * sqrt(Tqmin * (1.0 - 8.0 * u64)))) return 0.0f;
    const double err = (4.0 * s3 * eps * rmax * (1.0 + 0x1p-40) + 12.0 * eps * eps) * 1.0001;
    const double hw = (u * Tmax + 8.0 * u64 * Tmax + err + u * 60.1 * Ep * Ep) * (1.0 + 0x1p-30);
    int e;
    frexp((1.0 - 0x1p-22) / hw, &e);          // = f 2^e, f in [0.5, 1)
    const double kd = ldexp(1.0, e - 1);      // largest power of two <= (1 - 2^-22) / hw
    if (!(kd * (12.0 * Ep * Ep + 2.0 * Tmax) < 1e36) || !(2.0 * kd * Ep < 1e36)) return 0.0f;
    return (float)kd;
}

// ---------------------------------------------------------------------------
// Unit geometry: identical code in the descent and the walk kernels, so both
// derive bit-identical c, E and R'_u.
// ---------------------------------------------------------------------------
struct UnitGeom {
    int q0, nq, leaf;
    double lo[3], hi[3], c[3];
    double Ru, Ru2, Rx, E;  // R'_u, its square, the largest cull radius, the coordinate bound
    // this lane's queries (lane, lane + 32): fp64 coordinates, (2h)^2, caller index
    double qx[2], qy[2], qz[2], qT[2], qt[2];
    int32_t qo[2];
};

// rext: the largest cull radius of the unit's candidates (the gather walk:
// R'_u itself; the symmetric walk: the descent's rmax >= R'_u)
__device__ __forceinline__ void unit_setup(const WalkArgs &a, const int4 &UU, int lane, UnitGeom &G, double rext) {
    G.leaf = UU.x;
    G.q0 = UU.y;
    G.nq = UU.z;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    double Ru = 0.0;
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int k = lane + 32 * h;
        G.qx[h] = G.qy[h] = G.qz[h] = G.qT[h] = G.qt[h] = 0.0;
        G.qo[h] = 0;
        if (k < G.nq) {
            const double4 r = a.rec[G.q0 + k];
            const double t = __dmul_rn(2.0, a.h_tree[G.q0 + k]);  // 2h (exact)
            G.qx[h] = r.x;
            G.qy[h] = r.y;
            G.qz[h] = r.z;
            G.qT[h] = __dmul_rn(t, t);
            G.qt[h] = t;
            G.qo[h] = a.tree_order ? G.q0 + k : (int32_t)__double_as_longlong(r.w);
            // R' = 2h (1 + 2^-40) + 2^-50 M   (lemma L1/L2)
            Ru = fmax(Ru, __dadd_rn(__dmul_rn(t, 1.0 + 0x1p-40), __dmul_rn(0x1p-50, a.M)));
            lo[0] = fmin(lo[0], r.x); lo[1] = fmin(lo[1], r.y); lo[2] = fmin(lo[2], r.z);
            hi[0] = fmax(hi[0], r.x); hi[1] = fmax(hi[1], r.y); hi[2] = fmax(hi[2], r.z);
        }
    }
    // a unit holding its whole leaf has the leaf's tight box as its query box
    const bool whole = G.nq == a.leaf_count[G.leaf];
    const double *lb = a.leaf_box + 6 * (int64_t)G.leaf;
    double E = 0.0, Mu = 0.0;
    for (int l = 0; l < 3; l++) {
        G.lo[l] = whole ? lb[l] : warp_min(lo[l]);
        G.hi[l] = whole ? lb[3 + l] : warp_max(hi[l]);
        G.c[l] = 0.5 * (G.lo[l] + G.hi[l]);
        E = fmax(E, 0.5 * (G.hi[l] - G.lo[l]));
        Mu = fmax(Mu, fmax(fabs(G.lo[l]), fabs(G.hi[l])));
    }
    G.Ru = warp_max(Ru);
    G.Ru2 = __dmul_rn(G.Ru, G.Ru);
    G.Rx = fmax(G.Ru, rext);
    // a-priori bound |x - c| <= E per axis for queries and kept candidates (L4)
    G.E = (E + G.Rx) * 1.0001 + 4.0 * 0x1p-53 * Mu;
}

// The unit's query box and R'_u only (the descent): the same operations as
// unit_setup (min / max are exact and order independent), so both kernels
// see bit-identical boxes.  A whole-leaf unit needs only its queries' h.
__device__ __forceinline__ void unit_box(const WalkArgs &a, const int4 &UU, int lane, double (&lo)[3], double (&hi)[3],
                                         double &Ru, long long &hsum, bool &hbad) {
    const int q0 = UU.y, nq = UU.z;
    const bool whole = nq == a.leaf_count[UU.x];
    double r = 0.0;
    for (int l = 0; l < 3; l++) {
        lo[l] = INFINITY;
        hi[l] = -INFINITY;
    }
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int k = lane + 32 * h;
        if (k < nq) {
            double hv;
            if (a.h_src) {  // fused gather of h into tree order (+ validation, checksum: gather_h_kernel's)
                const int32_t i = a.tree_order ? q0 + k : a.perm[q0 + k];
                hv = a.h_src[i];
                a.h_out[q0 + k] = hv;
                hbad = hbad || !(hv > 0.0 && hv <= 1e150);
                hsum += __double_as_longlong(hv) * (2 * (long long)i + 1);
            } else {
                hv = a.h_tree[q0 + k];
            }
            const double t = __dmul_rn(2.0, hv);  // 2h (exact)
            r = fmax(r, __dadd_rn(__dmul_rn(t, 1.0 + 0x1p-40), __dmul_rn(0x1p-50, a.M)));
            if (!whole) {
                const double4 p = a.rec[q0 + k];
                lo[0] = fmin(lo[0], p.x); lo[1] = fmin(lo[1], p.y); lo[2] = fmin(lo[2], p.z);
                hi[0] = fmax(hi[0], p.x); hi[1] = fmax(hi[1], p.y); hi[2] = fmax(hi[2], p.z);
            }
        }
    }
    const double *lb = a.leaf_box + 6 * (int64_t)UU.x;
    for (int l = 0; l < 3; l++) {
        lo[l] = whole ? lb[l] : warp_min(lo[l]);
        hi[l] = whole ? lb[3 + l] : warp_max(hi[l]);
    }
    Ru = warp_max(r);
}

// x / d for d >= 1 (inv = fl32(1/d)): for x < 2^22 x is exact in fp32 and the
// rounded quotient is within one of the true one, fixed by one remainder
// test; larger x (a range of >= 2^22 cells of one node: huge b at tiny s,
// ADVICE r1) takes the exact integer division.
__device__ __forceinline__ unsigned small_div(unsigned x, unsigned d, float inv) {
    if (x >= (1u << 22)) return x / d;
    int q = __float2int_rz(__fmul_rn(__uint2float_rn(x), inv));
    const int r = (int)x - q * (int)d;
    q += (r < 0) ? -1 : ((r >= (int)d) ? 1 : 0);
    return (unsigned)q;
}

// Persistent warps claim work units in batches of consecutive (Morton-ordered,
// so spatially adjacent) units: one returning atomic per batch instead of one
// per unit on a single address, which serialised ~10^6 atomics per launch.
struct WorkBatch {
    long long next = 0, end = 0;
};
__device__ __forceinline__ long long next_unit(WorkBatch &w, long long *ctr, long long n, int batch, int lane) {
    if (w.next >= w.end) {
        long long b = 0;
        if (lane == 0) b = (long long)atomicAdd((unsigned long long *)ctr, (unsigned long long)batch);
        b = __shfl_sync(0xffffffffu, b, 0);
        w.next = b;
        w.end = b + batch < n ? b + batch : n;
    }
    return w.next < w.end ? w.next++ : n;
}

// Warp-uniform allocation from a per-warp slab [cur, end) refilled from a
// global counter; returns false when the arena capacity was exceeded.
struct Slab {
    long long cur = 0, end = 0;
};
__device__ __forceinline__ bool slab_reserve(Slab &s, long long need, long long chunk, long long cap, long long *ctr,
                                             int lane) {
    if (s.end - s.cur < need) {
        const long long size = need > chunk ? need : chunk;
        long long base = 0;
        if (lane == 0) base = (long long)atomicAdd((unsigned long long *)ctr, (unsigned long long)size);
        base = __shfl_sync(0xffffffffu, base, 0);
        s.cur = base;
        s.end = base + size;
    }
    return s.cur + need <= cap;
}

// ---------------------------------------------------------------------------
// desc_kernel: candidate-leaf lists (A10)
// ---------------------------------------------------------------------------
struct DescOut {
    int nleaf;
    long long loaded;
    bool overflow;  // a level frontier exceeded the frontier capacity
    double rmax;    // symmetric criterion: largest cull radius of a kept leaf
};

// R' of a particle (or of a subtree's largest h): 2h (1 + 2^-40) + 2^-50 M
// (lemma L1/L2); the same operations as the queries' R' in unit_box
__device__ __forceinline__ double rprime(double hh, double M) {
    return __dadd_rn(__dmul_rn(__dmul_rn(2.0, hh), 1.0 + 0x1p-40), __dmul_rn(0x1p-50, M));
}

// Breadth-first descent of one unit; appends the kept leaves to out[0, lim)
// (when out != nullptr) and returns how many there are.
// Internal-node cull (L3 for a whole subtree; the symmetric walk, where a
// far subtree of small h can be skipped -- for the gather walk the Eq. 5
// ranges prune as well and the extra loads did not pay): the child's equal-slice box
// [lo, lo + ext] contains its particles up to the rounding of the parent's
// Eq. 2 (a few ulps of |x - lo|), covered by the widening delta; the node is
// skipped only if that box is farther than R (1 + 2^-40) + delta from the
// query box, R = R'_u (gather) or max(R'_u, R'(h_max of the subtree))
// (symmetric).  Exact fp64 min / max, rounded products on a 2^-40 margin.
template <bool kSym>
__device__ __forceinline__ bool node_near(const WalkArgs &a, int32_t node, const double (&qlo)[3],
                                          const double (&qhi)[3], double Ru) {
    const NodeRec &nd = a.nodes[node];
    const double R = kSym ? fmax(Ru, rprime(a.node_hmax[node], a.M)) : Ru;
    double g2 = 0.0;
    for (int l = 0; l < 3; l++) {
        const double lo = nd.lo[l], hi = __dadd_rn(nd.lo[l], nd.ext[l]);
        const double d = (fabs(lo) + fabs(hi)) * 0x1p-40 + 0x1p-1000;
        const double g = fmax(0.0, fmax(__dsub_rn(__dsub_rn(lo, d), qhi[l]), __dsub_rn(qlo[l], __dadd_rn(hi, d))));
        g2 = __dadd_rn(g2, __dmul_rn(g, g));
    }
    const double Rc = __dadd_rn(__dmul_rn(R, 1.0 + 0x1p-40), 0x1p-1000);
    return g2 < __dmul_rn(Rc, Rc);
}

// kSym (symmetric criterion, R22): a node's Eq. 5 ranges use max(R'_u,
// R'(h_max of the node)) and a leaf is kept when its box is within max(R'_u,
// R'(h_max of the leaf)) of the query box: every j with d(i, j) below
// 2 max(h_i, h_j) (lemma L1) lies in a kept leaf.
template <bool kSym>
__device__ __forceinline__ DescOut descend(const WalkArgs &a, const double (&qlo)[3], const double (&qhi)[3],
                                           double Ru, int lane, int32_t *fcur, int32_t *fnext, long long fcap,
                                           int32_t *out, long long lim) {
    const double Ru2 = __dmul_rn(Ru, Ru);
    const unsigned lt = lanemask_lt();
    DescOut r{0, 0, false, Ru};
    long long loaded = 0;
    // leaf cell found by this lane: keep it if its tight box is within R'_u of
    // the query box (L3, exact fp64 box distance)
    auto emit = [&](bool is_leaf, int32_t leaf) {
        bool keep = false;
        if (is_leaf) {
            const double2 *lb = reinterpret_cast<const double2 *>(a.leaf_box + 6 * (int64_t)leaf);
            const double2 b0 = lb[0], b1 = lb[1], b2 = lb[2];  // lo x,y | lo z, hi x | hi y,z
            double gx = fmax(0.0, fmax(__dsub_rn(b0.x, qhi[0]), __dsub_rn(qlo[0], b1.y)));
            double gy = fmax(0.0, fmax(__dsub_rn(b0.y, qhi[1]), __dsub_rn(qlo[1], b2.x)));
            double gz = fmax(0.0, fmax(__dsub_rn(b1.x, qhi[2]), __dsub_rn(qlo[2], b2.y)));
            double g2 = __dadd_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)), __dmul_rn(gz, gz));
            if (kSym) {
                const double RL = fmax(Ru, rprime(a.leaf_hmax[leaf], a.M));
                keep = g2 < __dmul_rn(RL, RL);
                if (keep) r.rmax = fmax(r.rmax, RL);
            } else {
                keep = g2 < Ru2;
            }
        }
        const unsigned km = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const long long slot = r.nleaf + __popc(km & lt);
            if (out && slot < lim) out[slot] = leaf;
            loaded += a.leaf_count[leaf];
        }
        r.nleaf += __popc(km);
    };
    if (a.root_is_leaf) {
        emit(lane == 0, 0);
    } else {
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
                    const double Rn = kSym ? fmax(Ru, rprime(a.node_hmax[fcur[fi]], a.M)) : Ru;
                    int r0[3], r1[3];
                    for (int l = 0; l < 3; l++) {  // Eq. 5 with R'_u (lemma L2); b_z = nd.bz
                        const int bl = l == 2 ? nd.bz : b;
                        r0[l] = cell_coord_fast(__dsub_rn(qlo[l], Rn), nd.lo[l], nd.ext[l], nd.bx[l], bl);
                        r1[l] = cell_coord_fast(__dadd_rn(qhi[l], Rn), nd.lo[l], nd.ext[l], nd.bx[l], bl);
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
                        // cell offset inside the node's range (< b^3 < 2^32 for n < 2^31)
                        const unsigned local = (unsigned)(g - ostart);
                        const unsigned qx = small_div(local, onx, 1.0f / (float)onx);
                        const unsigned qy = small_div(qx, ony, 1.0f / (float)ony);
                        const int cx = ox + (int)(local - qx * onx);
                        const int cy = oy + (int)(qx - qy * ony);
                        const int cz = oz + (int)qy;
                        const long long j = cx + (long long)cy * ob + (long long)cz * ob * ob;  // Eq. 3
                        code = a.cells[ocb + j];
                        is_leaf = code >= 0;
                        is_node = code <= -2;
                        if (kSym && is_node) is_node = node_near<kSym>(a, code_node(code), qlo, qhi, Ru);
                        BT_DEV_CHECK(ocb + j < a.n_cells && code < a.n_leaves);
                    }
                    const unsigned nm = __ballot_sync(0xffffffffu, is_node);
                    const int slot = nnext + __popc(nm & lt);
                    if (is_node && slot < fcap) fnext[slot] = code_node(code);
                    nnext += __popc(nm);
                    emit(is_leaf, code);
                }
            }
            __syncwarp();
            if (nnext > fcap) {
                r.overflow = true;
                break;
            }
            int32_t *tmp = fcur;
            fcur = fnext;
            fnext = tmp;
            nf = nnext;
        }
    }
    for (int d = 16; d; d >>= 1) loaded += __shfl_xor_sync(0xffffffffu, loaded, d);
    r.loaded = loaded;
    if (kSym) r.rmax = warp_max(r.rmax);
    return r;
}

// The gather walk's unit geometry and query records (round 2, third pass:
// computed by the descent, which holds the unit's query box and R'_u already,
// instead of by the issue-bound walk): the same operations as unit_setup and
// the walk's setup -- c = (lo + hi) / 2, E, the band scale k = min over the
// queries of l4_band's (0 = force), per query (-2k a, fl32(k (|a|^2 - Mid)))
// with a = fl32(x - c), the fp32 query box and cull radius -- so the walk's
// decisions are bit-identical either way.
__device__ __forceinline__ void prep_gather_unit(const WalkArgs &a, const int4 &UU, long long uid, int lane,
                                                 const double (&lo)[3], const double (&hi)[3], double Ru) {
    const int q0 = UU.y, nq = UU.z;
    double c[3], E = 0.0, Mu = 0.0;
    for (int l = 0; l < 3; l++) {
        c[l] = 0.5 * (lo[l] + hi[l]);
        E = fmax(E, 0.5 * (hi[l] - lo[l]));
        Mu = fmax(Mu, fmax(fabs(lo[l]), fabs(hi[l])));
    }
    E = (E + Ru) * 1.0001 + 4.0 * 0x1p-53 * Mu;  // (Rx = R'_u: the gather walk)
    const double eps = l4_eps(E);
    float kq[2] = {INFINITY, INFINITY}, mid[2] = {0.0f, 0.0f};
    float ax[2] = {0.f, 0.f}, ay[2] = {0.f, 0.f}, az[2] = {0.f, 0.f};
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int k = lane + 32 * h;
        if (k < nq) {
            const double4 r = a.rec[q0 + k];  // (reloaded: values kept from unit_box cost the descent registers)
            const double t = __dmul_rn(2.0, a.h_tree[q0 + k]);  // 2h (exact)
            l4_band(__dmul_rn(t, t), t, E, eps, a.exact_only != 0, kq[h], mid[h]);
            ax[h] = __double2float_rn(__dsub_rn(r.x, c[0]));
            ay[h] = __double2float_rn(__dsub_rn(r.y, c[1]));
            az[h] = __double2float_rn(__dsub_rn(r.z, c[2]));
        }
    }
    float ku = fminf(kq[0], kq[1]);
    for (int d = 16; d; d >>= 1) ku = fminf(ku, __shfl_xor_sync(0xffffffffu, ku, d));
    const bool force = ku == 0.0f;
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int k = lane + 32 * h;
        if (k < nq) {
            const float m2k = -2.0f * ku;
            const double qq = (double)ax[h] * ax[h] + (double)ay[h] * ay[h] + (double)az[h] * az[h];
            const float bq = force ? 0.0f : __double2float_rn((double)ku * (qq - (double)mid[h]));
            a.qrec[q0 + k] = make_float4(m2k * ax[h], m2k * ay[h], m2k * az[h], bq);
        }
    }
    if (lane == 0) {
        float blo[3], bhi[3];
        for (int l = 0; l < 3; l++) {
            blo[l] = __double2float_rn(__dsub_rn(lo[l], c[l]));
            bhi[l] = __double2float_rn(__dsub_rn(hi[l], c[l]));
        }
        const double rc = (Ru + 4.0 * eps) * (1.0 + 0x1p-20);
        const double rc2 = rc * rc * (1.0 + 0x1p-40);
        UnitPrep P;
        P.c[0] = c[0];
        P.c[1] = c[1];
        P.c[2] = c[2];
        P.E = E;
        P.box0 = make_float4(blo[0], blo[1], blo[2], (rc2 < 3.0e38) ? __double2float_ru(rc2) : INFINITY);
        P.box1 = make_float4(bhi[0], bhi[1], bhi[2], 0.0f);
        P.k = ku;
        P.pad = 0;
        a.uprep[uid] = P;
    }
}

// exact arena bounds of the walk (a unit stages at most `loaded` candidates),
// summed per warp (lane 0) and added once per warp at the end of the pass
// (two same-address atomics per unit cost the cfg 2 descent 0.18 -> 0.13 ms)
struct Need {
    unsigned long long c = 0, m = 0;
    __device__ void add(long long loaded, int nq) {
        c += (unsigned long long)loaded;
        m += (unsigned long long)(((loaded + 63) >> 6) * nq);
    }
    __device__ void flush(const WalkArgs &a) const {
        if (c) atomicAdd((unsigned long long *)&a.ctr[C_NEEDC], c);
        if (m) atomicAdd((unsigned long long *)&a.ctr[C_NEEDM], m);
    }
};

// kBig = false: frontier in shared memory, list from per-warp slabs with at
//   most kListReserve leaves per unit; a unit exceeding either is marked
//   (nleaf = -1) for the big pass.
// kBig = true: only marked units; frontier in global scratch (front_cap =
//   all nodes), the list counted first and allocated exactly.
// (A batched variant -- one descent with the union box of 8 Morton-adjacent
// units, each unit filtering the union list -- measured slower in round 2:
// cfg 5 descent 2.9 -> 5.5 ms, the union lists being far larger than a unit's.)
template <bool kBig, bool kSym>
__global__ void __launch_bounds__(kDescThreads) desc_kernel(WalkArgs a) {
    __shared__ int32_t sfront[kBig ? 1 : kDescThreads / 32][2][kBig ? 1 : kFrontCap];
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int32_t *f0, *f1;
    long long fcap;
    if (kBig) {
        f0 = a.front + gwarp * 2 * a.front_cap;
        f1 = f0 + a.front_cap;
        fcap = a.front_cap;
    } else {
        f0 = sfront[threadIdx.x >> 5][0];
        f1 = sfront[threadIdx.x >> 5][1];
        fcap = kFrontCap;
    }
    Slab ls;
    WorkBatch wb;
    Need need;
    long long hsum = 0;  // fused gather of h (first pass only): checksum and validity of this lane's values
    bool hbad = false;
    for (;;) {
        const long long uid = next_unit(wb, &a.ctr[kBig ? C_WORK4 : C_WORK], a.n_units, kBig ? 1 : a.desc_batch, lane);
        if (uid >= a.n_units) break;
        if (kBig && a.urun[uid].nleaf >= 0) continue;
        const int4 U = a.units[uid];
        double qlo[3], qhi[3], Ru;
        unit_box(a, U, lane, qlo, qhi, Ru, hsum, hbad);
        if (!kBig && !kSym && a.uprep) prep_gather_unit(a, U, uid, lane, qlo, qhi, Ru);
        UnitRun &R = a.urun[uid];
        if (!kBig) {
            const bool ok = slab_reserve(ls, kListReserve, kListSlab, a.list_cap, &a.ctr[C_LIST], lane);
            const long long lim = ls.end - ls.cur;
            DescOut d = descend<kSym>(a, qlo, qhi, Ru, lane, f0, f1, fcap, ok ? a.ulist + ls.cur : nullptr, lim);
            const bool fits = ok && !d.overflow && d.nleaf <= lim;
            if (lane == 0) {
                R.list_off = ls.cur;
                R.nleaf = fits ? d.nleaf : -1;
                R.loaded = (int)d.loaded;
                R.rmax = d.rmax;
                if (!fits) atomicAdd((unsigned long long *)&a.ctr[C_BIG], 1ull);
                else need.add(d.loaded, U.z);
            }
            if (fits) ls.cur += d.nleaf;
        } else {
            DescOut d = descend<kSym>(a, qlo, qhi, Ru, lane, f0, f1, fcap, nullptr, 0);
            long long base = 0;
            if (lane == 0) base = (long long)atomicAdd((unsigned long long *)&a.ctr[C_LIST], (unsigned long long)d.nleaf);
            base = __shfl_sync(0xffffffffu, base, 0);
            const bool ok = !d.overflow && base + d.nleaf <= a.list_cap;
            if (ok) descend<kSym>(a, qlo, qhi, Ru, lane, f0, f1, fcap, a.ulist + base, d.nleaf);
            if (lane == 0) {
                R.list_off = base;
                R.nleaf = ok ? d.nleaf : -2;  // -2: list arena too small (host grows it and redoes the pass)
                R.loaded = (int)d.loaded;
                R.rmax = d.rmax;
                need.add(d.loaded, U.z);
            }
        }
        __syncwarp();
    }
    if (lane == 0) need.flush(a);
    if (a.h_src) {
        for (int d = 16; d; d >>= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, d);
        const bool bad = __any_sync(0xffffffffu, hbad);
        if (lane == 0) {
            atomicAdd((unsigned long long *)&a.ctr[C_HSUM], (unsigned long long)hsum);
            if (bad) atomicOr((unsigned long long *)&a.ctr[C_HBAD], 1ull);
        }
    }
}

// ---------------------------------------------------------------------------
// walk_kernel: staging + pair tests (A10, A11)
// ---------------------------------------------------------------------------
struct UnitSm {                     // per-warp unit state (shared memory)
    long long cand_base, mask_base;  // the unit's record bases
    Slab cs, ms;                     // the warp's candidate / mask slabs
    long long tests, exact, staged, loaded, nzw;  // warp totals
    int32_t *cand_ptr;               // the unit's candidate-index records (a.cands + cand_base)
    double c[3], E;                  // unit centre, coordinate bound (L4)
    double Ru, eps, tqmin;           // symmetric: R'_u, l4_eps(E), smallest query threshold
    float4 box0, box1;               // fp32 query box relative to c: (lo xyz, cull2), (hi xyz, -)
    int q0, nq;                      // (8-byte aligned: read as one int2)
    float k;                         // band scale of the unit (power of two; 0: force)
    int rec_ok, force;
};

struct WalkSmem {
    float4 q0[kQ + 1];              // ax, ax, ay, ay  (fp32, relative to the unit centre)
    float4 q1[kQ + 1];              // az, az, c, c   (band map d' = s k + c); [kQ]: look-ahead pad
    int self[kQ];                   // unit slot of each query's own record (-1: none)
    unsigned long long mask[kQ][2]; // the block's neighbor masks [query][chunk] (one 16-B store per query)
    int ldel[kGroup];               // group leaves: first tree position - exclusive prefix of counts
    unsigned lstart[kGroupPos / 32];       // group positions: bit p set where a leaf starts (p = 32 w + bit)
    unsigned char lwpre[kGroupPos / 32];   // leaves starting before word w
    float4 loff[kGroup];            // group leaves: fl32(c_leaf - c), w = 1 compact / 0 fp64 records
    float lcull[kGroup];            // symmetric: group leaves' fp32 cull radius^2 (max(R'_u, R'(h_max)))
    float2 qm[kQ + 1];              // symmetric: -k Mid_i per query (packed pair); [kQ]: look-ahead pad
    float4 stg[kStg];               // staged candidates: fp32 x, y, z relative to the unit centre, tree position
    UnitSm u;
};

// density mode (consumer fusion): per-query 1/h and the
// block's candidates with their masses
template <bool kDensity>
struct DensitySm {};
template <>
struct DensitySm<true> {
    float hinv[kQ];
    float4 qraw[kQ];  // fp32 query coordinates relative to the unit centre
};
template <bool kDensity, bool kSym>
struct WalkSmemT : WalkSmem {
    DensitySm<kDensity> d;
};

// fp32 square root on the SFU (sqrt.approx: relative error ~2^-22, sqrt(0) = 0)
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));  // (flushing a subnormal r^2 gives r = 0: w(0), the limit)
    return r;
}

// The exact band of lemma L4 (rare): recompute the block's pairs with the
// hot loop's fp32 operations and let the fp64 predicate decide every pair
// with |d'| <= 1 (all pairs when `force`; padding slots >= n are never
// neighbors).  blk: the block's staged candidates (ax, ay, az, tree position).
// symmetric criterion: the candidate threshold term -k Mid_j of a staged
// candidate (tree position tp), +inf when it cannot decide (Tj <= Tqmin, L4s)
__device__ __forceinline__ float cand_thr(const WalkArgs &a, const UnitSm &u, int tp) {
    const double tj = __dmul_rn(2.0, a.h_tree[tp]);
    const double Tj = __dmul_rn(tj, tj);
    return Tj > u.tqmin ? -u.k * __double2float_rn(Tj) : __int_as_float(0x7f800000);
}

template <bool kSym>
__device__ __noinline__ void resolve_band(WalkSmemT<false, kSym> &S, const WalkArgs &a, int lane, int b0, int n,
                                          long long &exact) {
    const float4 *blk = S.stg + b0;
    const int nch = (n + 63) >> 6;
    const float inf = __int_as_float(0x7f800000);
    const float ku = S.u.k;
    const bool force = S.u.force != 0;  // (inf used for padding Ac)
    const int q0 = S.u.q0, nq = S.u.nq;
    for (int k = 0; k < nch; k++) {
        float4 c[2];
        float ac[2], nk[2] = {0.f, 0.f};
        bool real[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int s = 64 * k + 32 * h + lane;
            real[h] = s < n;
            c[h] = real[h] ? blk[s] : make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
            const float nc = __fmaf_rn(c[h].z, c[h].z, __fmaf_rn(c[h].y, c[h].y, __fmul_rn(c[h].x, c[h].x)));
            ac[h] = real[h] ? __fmul_rn(ku, nc) : inf;  // identical to test_block
            if constexpr (kSym) nk[h] = real[h] ? cand_thr(a, S.u, __float_as_int(c[h].w)) : 0.f;
        }
        for (int q = 0; q < nq; q++) {
            const float4 Q0 = S.q0[q], Q1 = S.q1[q];
            bool flag[2];
#pragma unroll
            for (int h = 0; h < 2; h++) {
                // the hot loop's v, operation for operation
                const float v = __fmaf_rn(c[h].x, Q0.x, __fmaf_rn(c[h].y, Q0.z, __fmaf_rn(c[h].z, Q1.x, __fadd_rn(ac[h], Q1.z))));
                if (kSym) {
                    const float w = __fadd_rn(v, fminf(S.qm[q].x, nk[h]));  // the hot loop's min(v_i, v_j)
                    flag[h] = real[h] && (force || fabsf(w) <= 1.0f);
                } else {
                    flag[h] = real[h] && (force || fabsf(v) <= 1.0f);
                }
            }
            const unsigned f0 = __ballot_sync(0xffffffffu, flag[0]), f1 = __ballot_sync(0xffffffffu, flag[1]);
            if (!(f0 | f1)) continue;
            const int qp = q0 + q;
            const double4 Qr = a.rec[qp];
            const double t = __dmul_rn(2.0, a.h_tree[qp]);
            const double T = __dmul_rn(t, t);
            bool e[2] = {false, false};
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int tp = __float_as_int(c[h].w);
                if (flag[h] && tp != qp) {
                    double Tp = T;
                    if (kSym) {  // the pair's threshold: fl((2 max(h_i, h_j))^2) = max(T_i, T_j)
                        const double tj = __dmul_rn(2.0, a.h_tree[tp]);
                        Tp = fmax(T, __dmul_rn(tj, tj));
                    }
                    e[h] = exact_pair(Qr.x, Qr.y, Qr.z, Tp, a.rec[tp]);
                }
            }
            const unsigned m0 = __ballot_sync(0xffffffffu, e[0]), m1 = __ballot_sync(0xffffffffu, e[1]);
            if (lane == 0) {
                const unsigned long long fm = ((unsigned long long)f1 << 32) | f0;
                const unsigned long long em = ((unsigned long long)m1 << 32) | m0;
                S.mask[q][k] = (S.mask[q][k] & ~fm) | em;
            }
            exact += __popc(f0) + __popc(f1);
            __syncwarp();
        }
    }
    __syncwarp();
}

// The band by candidate (round 2, third pass): the lanes in fl own every
// candidate with a banded pair (a lane's bmin covers its four candidates and
// all queries), so only their candidates are redone -- each broadcast to the
// lanes, lanes = queries, with the hot loop's fp32 operations -- and the
// pairs with |v| <= 1 (symmetric: |w| <= 1) decided by the fp64 predicate.
// Not for `force` (every pair exact): resolve_band.
#ifndef BT_BAND_LANES
#define BT_BAND_LANES 4
#endif
constexpr int kBandLanes = BT_BAND_LANES;
template <bool kSym>
__device__ __noinline__ void resolve_band_lanes(WalkSmemT<false, kSym> &S, const WalkArgs &a, int lane, int b0, int n,
                                                unsigned fl, long long &exact) {
    const float ku = S.u.k;
    const int q0 = S.u.q0, nq = S.u.nq;
    int nex = 0;  // this lane's exact pairs (summed over the warp at the end)
    while (fl) {
        const int l = __ffs(fl) - 1;
        fl &= fl - 1;
#pragma unroll 1
        for (int j = 0; j < 4; j++) {
            const int s = 32 * j + l;  // block slot of the lane's j-th candidate
            if (s >= n) break;
            const float4 c = S.stg[b0 + s];
            const float nc = __fmaf_rn(c.z, c.z, __fmaf_rn(c.y, c.y, __fmul_rn(c.x, c.x)));
            const float ac = __fmul_rn(ku, nc);  // identical to test_block
            const int tp = __float_as_int(c.w);
            float nkc = 0.f;
            if constexpr (kSym) nkc = cand_thr(a, S.u, tp);
            const unsigned long long bit = 1ull << (s & 63);
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int q = lane + 32 * h;
                if (q >= nq) continue;
                const float4 Q0 = S.q0[q], Q1 = S.q1[q];
                // the hot loop's v, operation for operation
                const float v = __fmaf_rn(c.x, Q0.x, __fmaf_rn(c.y, Q0.z, __fmaf_rn(c.z, Q1.x, __fadd_rn(ac, Q1.z))));
                const float w = kSym ? __fadd_rn(v, fminf(S.qm[q].x, nkc)) : v;
                if (!(fabsf(w) <= 1.0f)) continue;
                const int qp = q0 + q;
                bool e = false;
                if (tp != qp) {
                    const double t = __dmul_rn(2.0, a.h_tree[qp]);
                    double T = __dmul_rn(t, t);
                    if (kSym) {  // the pair's threshold: fl((2 max(h_i, h_j))^2) = max(T_i, T_j)
                        const double tj = __dmul_rn(2.0, a.h_tree[tp]);
                        T = fmax(T, __dmul_rn(tj, tj));
                    }
                    const double4 Qr = a.rec[qp];
                    e = exact_pair(Qr.x, Qr.y, Qr.z, T, a.rec[tp]);
                }
                unsigned long long &mw = S.mask[q][s >> 6];
                mw = e ? (mw | bit) : (mw & ~bit);
                nex++;
            }
        }
    }
    exact += __reduce_add_sync(0xffffffffu, (unsigned)nex);
    __syncwarp();
}

// Density mode (reading R21), round 2: the SPH sum needs
// no neighbor masks.  The M4 shape vanishes at the support's edge (w(2) = 0,
// w(2 - d) = d^3 / 4), so a pair decided differently by fp32 near r = 2h
// changes rho by ~(its distance to the edge)^3 -- nothing at fp32 precision;
// w(q) = max(0, 2 - q)^3 / 4 - max(0, 1 - q)^3 is the spline on both
// pieces and 0 beyond, branch-free.  So every staged candidate is summed
// against every query of the unit: lanes = queries (balanced: each lane owns
// one query's sum; the self pair gives w(0) = 1, the m_i W(0, h_i) term),
// candidates broadcast from shared memory in packed pairs, the arithmetic in
// packed f32x2.
__device__ __forceinline__ unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ void density_block(WalkSmemT<true, false> &S, const WalkArgs &a, int lane, int b0, int n,
                                              double (&dacc)[2]) {
    const float4 *blk = S.stg + b0;
    // the block's candidates with their masses, repacked in place over
    // stg[0, kBlk) (read into registers first; a second block, b0 = kBlk,
    // lies beyond the packed range)
    float4 *P = S.stg;                // pair p: (x_2p, x_2p+1, y_2p, y_2p+1)
    float4 *Qz = S.stg + kBlk / 2;    // pair p: (z_2p, z_2p+1, m_2p, m_2p+1)
    float *Pf = reinterpret_cast<float *>(P), *Qf = reinterpret_cast<float *>(Qz);
    float4 cc[4];
    float mm[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const int sl = 32 * j + lane;
        cc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        mm[j] = 0.f;  // padding: m = 0 (no contribution)
        if (sl < n) {
            cc[j] = blk[sl];
            mm[j] = (float)a.m_tree[__float_as_int(cc[j].w)];
        }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const int sl = 32 * j + lane;
        const float4 c = cc[j];
        const float m = mm[j];
        const int p = sl >> 1, o = sl & 1;
        Pf[4 * p + o] = c.x;
        Pf[4 * p + 2 + o] = c.y;
        Qf[4 * p + o] = c.z;
        Qf[4 * p + 2 + o] = m;
    }
    __syncwarp();
    const int nq = S.u.nq, np = (n + 1) >> 1;
    const unsigned long long two = pk(2.0f, 2.0f), mone = pk(-1.0f, -1.0f), mfour = pk(-4.0f, -4.0f);
#pragma unroll 1
    for (int h = 0; h < 2; h++) {
        if (32 * h >= nq) break;  // (warp-uniform)
        const int q = lane + 32 * h;
        const float4 qr = S.d.qraw[q < nq ? q : 0];
        const float hv = S.d.hinv[q < nq ? q : 0];
        const unsigned long long nqx = pk(-qr.x, -qr.x), nqy = pk(-qr.y, -qr.y), nqz = pk(-qr.z, -qr.z);
        const unsigned long long nhinv = pk(-hv, -hv);
        unsigned long long acc = 0ull;  // (+0, +0): sum of m_j (4 w(q_ij))
#pragma unroll 4
        for (int p = 0; p < np; p++) {
            const float4 A = P[p], B = Qz[p];
            const unsigned long long dx = f2_add(pk(A.x, A.y), nqx), dy = f2_add(pk(A.z, A.w), nqy),
                                     dz = f2_add(pk(B.x, B.y), nqz);
            const unsigned long long r2 = f2_fma(dz, dz, f2_fma(dy, dy, f2_mul(dx, dx)));
            const unsigned long long nq2 = f2_mul(pk(sqrt_approx(lo_f(r2)), sqrt_approx(hi_f(r2))), nhinv);  // -r / h
            const unsigned long long t2 = f2_add(two, nq2);   // 2 - q
            const unsigned long long t1 = f2_add(t2, mone);   // 1 - q
            const unsigned long long u2 = pk(fmaxf(lo_f(t2), 0.f), fmaxf(hi_f(t2), 0.f));
            const unsigned long long u1 = pk(fmaxf(lo_f(t1), 0.f), fmaxf(hi_f(t1), 0.f));
            const unsigned long long c2 = f2_mul(f2_mul(u2, u2), u2), c1 = f2_mul(f2_mul(u1, u1), u1);
            acc = f2_fma(pk(B.z, B.w), f2_fma(c1, mfour, c2), acc);  // m (max(0,2-q)^3 - 4 max(0,1-q)^3)
        }
        if (q < nq) dacc[h] += 0.25 * ((double)lo_f(acc) + (double)hi_f(acc));  // w = (...) / 4
    }
    __syncwarp();
}

// query loop unroll of the gather pair tests (queries padded to a multiple)
#ifndef BT_TEST_UNROLL
#define BT_TEST_UNROLL 2
#endif
constexpr int kTestUnroll = BT_TEST_UNROLL;
// units with at least BT_FUNNEL_Q queries record masks by funnel shifts (65: none)
#ifndef BT_FUNNEL_Q
#define BT_FUNNEL_Q 65
#endif
constexpr int kFunnelQ = BT_FUNNEL_Q;

// Test n (<= kBlk) staged candidates (blk, unit slots us0 .. us0 + n) against
// the unit's queries and record the block's masks; returns this lane's count
// increments for queries (lane, lane + 32).
template <bool kDensity, bool kSym>
__device__ __forceinline__ int2 test_block(WalkSmemT<kDensity, kSym> &S, const WalkArgs &a, int lane, int n, int us0,
                                           int b0, double (&dacc)[2]) {
    const float4 *blk = S.stg + b0;
    const float inf = __int_as_float(0x7f800000);
    const int nch = (n + 63) >> 6;  // 1 or 2 chunks of 64
    const int nq = S.u.nq;
    // this lane's candidates: chunk 0 -> slots (l, l + 32), chunk 1 -> (l + 64, l + 96);
    // padding slots: c = 0, Ac = +inf (v = +inf: never a neighbor, never banded)
    const float ku = S.u.k;
    float4 c[4];
    float ac[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const int s = 32 * j + lane;
        c[j] = (s < n) ? blk[s] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float nc = __fmaf_rn(c[j].z, c[j].z, __fmaf_rn(c[j].y, c[j].y, __fmul_rn(c[j].x, c[j].x)));
        ac[j] = (s < n) ? __fmul_rn(ku, nc) : inf;  // k |c|^2 (exact scaling)
    }
    const unsigned long long xa = pk(c[0].x, c[1].x), ya = pk(c[0].y, c[1].y), za = pk(c[0].z, c[1].z),
                             aa = pk(ac[0], ac[1]);
    const unsigned long long xb = pk(c[2].x, c[3].x), yb = pk(c[2].y, c[3].y), zb = pk(c[2].z, c[3].z),
                             ab = pk(ac[2], ac[3]);
    const int nqp = (nq + 1) & ~1;  // padded to even (the pad query never matches)
    // the gather loops: padded to a multiple of their unroll (pad queries never match)
    const int nqu = (nq + kTestUnroll - 1) / kTestUnroll * kTestUnroll;
    // shared addresses of the query records (two LDS.128 per query)
    const unsigned aq0 = (unsigned)__cvta_generic_to_shared(&S.q0[0]);
    const unsigned aq1 = (unsigned)__cvta_generic_to_shared(&S.q1[0]);
    float bmin = 2.0f;  // min |v| over the block's pairs: <= 1 -> some pair is banded
    // query records (-2k q, k(|q|^2 - Mid)), loaded one query ahead of their use (LDS latency)
    auto ldq = [&](int q, float4 &Q0, float4 &Q1) {
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(Q0.x), "=f"(Q0.y), "=f"(Q0.z), "=f"(Q0.w) : "r"(aq0 + 16 * q));
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(Q1.x), "=f"(Q1.y), "=f"(Q1.z), "=f"(Q1.w) : "r"(aq1 + 16 * q));
    };
    float4 N0, N1;
    ldq(0, N0, N1);
    if constexpr (kSym) {
        // symmetric criterion (lemma L4s): u = k |c - q|^2 without Mid, then
        // v_i = u - k Mid_i (query threshold) and v_j = u - k Mid_j (candidate
        // threshold, +inf when it cannot decide); the bit is w < 0 for
        // w = min(v_i, v_j) = u + min(-k Mid_i, -k Mid_j), and only |w| <= 1
        // is uncertain (w < -1: one threshold certainly holds; w > 1: neither)
        float nk[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int sl = 32 * j + lane;
            nk[j] = (sl < n) ? cand_thr(a, S.u, __float_as_int(c[j].w)) : inf;  // (padding: u = +inf anyway)
        }
        const unsigned aqm = (unsigned)__cvta_generic_to_shared(&S.qm[0]);
        unsigned long long NM;
        asm volatile("ld.shared.b64 %0, [%1];" : "=l"(NM) : "r"(aqm));
        // a block whose every candidate threshold cannot decide (all +inf: the
        // common case inside a region of one h) tests the query thresholds alone
        const bool red = __all_sync(0xffffffffu, nk[0] == inf && nk[1] == inf && nk[2] == inf && nk[3] == inf);
        // (four loop variants -- all thresholds or query thresholds only, two
        // chunks or one -- so no branch sits inside a loop with ballots)
#define BT_SYM_LOOP(TWO, RED)                                                                                    \
    for (int q = 0; q < nqp; q++) {                                                                              \
        const float4 Q0 = N0, Q1 = N1;                                                                           \
        const unsigned long long qm = NM;                                                                        \
        ldq(q + 1, N0, N1);                                                                                      \
        asm volatile("ld.shared.b64 %0, [%1];" : "=l"(NM) : "r"(aqm + 8 * (q + 1)));                          \
        const unsigned long long qx = pk(Q0.x, Q0.y), qy = pk(Q0.z, Q0.w), qz = pk(Q1.x, Q1.y),                 \
                                 bq = pk(Q1.z, Q1.w);                                                            \
        const unsigned long long ua = f2_fma(xa, qx, f2_fma(ya, qy, f2_fma(za, qz, f2_add(aa, bq))));           \
        /* w = u + min(-k Mid_i, -k Mid_j) = min(v_i, v_j) (fl(u + .) is monotone) */                            \
        const unsigned long long wa = f2_add(ua, RED ? qm : pk(fminf(lo_f(qm), nk[0]), fminf(lo_f(qm), nk[1])));  \
        bmin = fminf(bmin, fminf(fabsf(lo_f(wa)), fabsf(hi_f(wa))));                                             \
        unsigned m2 = 0u, m3 = 0u;                                                                               \
        const unsigned m0 = __ballot_sync(0xffffffffu, lo_f(wa) < 0.0f);                                         \
        const unsigned m1 = __ballot_sync(0xffffffffu, hi_f(wa) < 0.0f);                                         \
        if (TWO) {                                                                                               \
            const unsigned long long ub = f2_fma(xb, qx, f2_fma(yb, qy, f2_fma(zb, qz, f2_add(ab, bq))));       \
            const unsigned long long wb =                                                                        \
                f2_add(ub, RED ? qm : pk(fminf(lo_f(qm), nk[2]), fminf(lo_f(qm), nk[3])));                       \
            bmin = fminf(bmin, fminf(fabsf(lo_f(wb)), fabsf(hi_f(wb))));                                         \
            m2 = __ballot_sync(0xffffffffu, lo_f(wb) < 0.0f);                                                    \
            m3 = __ballot_sync(0xffffffffu, hi_f(wb) < 0.0f);                                                    \
        }                                                                                                        \
        if (lane == 0)                                                                                           \
            *reinterpret_cast<ulonglong2 *>(S.mask[q]) =                                                         \
                make_ulonglong2(((unsigned long long)m1 << 32) | m0, ((unsigned long long)m3 << 32) | m2);      \
    }
        if (nch == 2) {
            if (red) {
#pragma unroll 2
                BT_SYM_LOOP(true, true)
            } else {
#pragma unroll 2
                BT_SYM_LOOP(true, false)
            }
        } else {
            if (red) {
#pragma unroll 2
                BT_SYM_LOOP(false, true)
            } else {
#pragma unroll 2
                BT_SYM_LOOP(false, false)
            }
        }
#undef BT_SYM_LOOP
    } else if (nq >= kFunnelQ) {
        // (BT_FUNNEL_Q, off by default) masks by funnel shifts: the sign bit of
        // each v shifted into a per-candidate word over up to 32 queries, then a
        // 32 x 32 bit transpose (five shuffle rounds) so that lane q holds query
        // q's ballot words.  Fewer instructions per query than four compares and
        // ballots but ~40 per transpose: measured slower at cfg 5 (walk 17.6 ms
        // with BT_FUNNEL_Q = 16 vs 15.5).  Compiled in, it also changes the
        // register allocation of the ballot loops below: their 4 ballots land in
        // the STS.128 quad directly (25 instead of 27.5 SASS per query; walk
        // 15.85 -> 15.46 ms at cfg 5).
        auto funnel = [&](auto two_chunks) {
            constexpr bool kTwo = decltype(two_chunks)::value;
            unsigned acc[4] = {0u, 0u, 0u, 0u};
            for (int qb = 0; qb < nqp; qb += 32) {
                const int qe = min(qb + 32, nqp);
#pragma unroll 2
                for (int q = qb; q < qe; q++) {
                    const float4 Q0 = N0, Q1 = N1;
                    ldq(q + 1, N0, N1);
                    const unsigned long long qx = pk(Q0.x, Q0.y), qy = pk(Q0.z, Q0.w), qz = pk(Q1.x, Q1.y),
                                             bq = pk(Q1.z, Q1.w);
                    const unsigned long long da = f2_fma(xa, qx, f2_fma(ya, qy, f2_fma(za, qz, f2_add(aa, bq))));
                    acc[0] = __funnelshift_l(__float_as_uint(lo_f(da)), acc[0], 1);
                    acc[1] = __funnelshift_l(__float_as_uint(hi_f(da)), acc[1], 1);
                    if constexpr (kTwo) {
                        const unsigned long long db =
                            f2_fma(xb, qx, f2_fma(yb, qy, f2_fma(zb, qz, f2_add(ab, bq))));
                        bmin = fminf(fminf(bmin, fminf(fabsf(lo_f(da)), fabsf(hi_f(da)))),
                                     fminf(fabsf(lo_f(db)), fabsf(hi_f(db))));
                        acc[2] = __funnelshift_l(__float_as_uint(lo_f(db)), acc[2], 1);
                        acc[3] = __funnelshift_l(__float_as_uint(hi_f(db)), acc[3], 1);
                    } else {
                        bmin = fminf(bmin, fminf(fabsf(lo_f(da)), fabsf(hi_f(da))));
                    }
                }
                const int sh = 32 - (qe - qb);
                unsigned w[4];
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    unsigned x = __brev(acc[j]) >> sh;
                    const unsigned masks[5] = {0x0000ffffu, 0x00ff00ffu, 0x0f0f0f0fu, 0x33333333u, 0x55555555u};
#pragma unroll
                    for (int r = 0; r < 5; r++) {
                        const int s2 = 16 >> r;
                        const unsigned m = masks[r];
                        const unsigned y = __shfl_xor_sync(0xffffffffu, x, s2);
                        x = (lane & s2) ? ((x & ~m) | ((y >> s2) & m)) : ((x & m) | ((y << s2) & ~m));
                    }
                    w[j] = x;
                }
                if (lane < qe - qb) {
                    if (kTwo)
                        *reinterpret_cast<ulonglong2 *>(S.mask[qb + lane]) = make_ulonglong2(
                            ((unsigned long long)w[1] << 32) | w[0], ((unsigned long long)w[3] << 32) | w[2]);
                    else
                        S.mask[qb + lane][0] = ((unsigned long long)w[1] << 32) | w[0];
                }
            }
        };
        if (nch == 2) funnel(std::true_type{});
        else funnel(std::false_type{});
    } else if (nch == 2) {
#pragma unroll kTestUnroll
        for (int q = 0; q < nqu; q++) {
            const float4 Q0 = N0, Q1 = N1;
            ldq(q + 1, N0, N1);  // q + 1 <= nqu <= 64: within the padded arrays
            const unsigned long long qx = pk(Q0.x, Q0.y), qy = pk(Q0.z, Q0.w), qz = pk(Q1.x, Q1.y),
                                     bq = pk(Q1.z, Q1.w);
            // v = k (|c - q|^2 - Mid) expanded: one add + three FMA per packed pair (lemma L4)
            const unsigned long long da = f2_fma(xa, qx, f2_fma(ya, qy, f2_fma(za, qz, f2_add(aa, bq))));
            const unsigned long long db = f2_fma(xb, qx, f2_fma(yb, qy, f2_fma(zb, qz, f2_add(ab, bq))));
            bmin = fminf(fminf(bmin, fminf(fabsf(lo_f(da)), fabsf(hi_f(da)))), fminf(fabsf(lo_f(db)), fabsf(hi_f(db))));
            const unsigned m0 = __ballot_sync(0xffffffffu, lo_f(da) < 0.0f);
            const unsigned m1 = __ballot_sync(0xffffffffu, hi_f(da) < 0.0f);
            const unsigned m2 = __ballot_sync(0xffffffffu, lo_f(db) < 0.0f);
            const unsigned m3 = __ballot_sync(0xffffffffu, hi_f(db) < 0.0f);
            if (lane == 0) {
                *reinterpret_cast<ulonglong2 *>(S.mask[q]) =
                    make_ulonglong2(((unsigned long long)m1 << 32) | m0, ((unsigned long long)m3 << 32) | m2);
            }
        }
    } else {
#pragma unroll kTestUnroll
        for (int q = 0; q < nqu; q++) {
            const float4 Q0 = N0, Q1 = N1;
            ldq(q + 1, N0, N1);
            const unsigned long long qx = pk(Q0.x, Q0.y), qy = pk(Q0.z, Q0.w), qz = pk(Q1.x, Q1.y),
                                     bq = pk(Q1.z, Q1.w);
            const unsigned long long da = f2_fma(xa, qx, f2_fma(ya, qy, f2_fma(za, qz, f2_add(aa, bq))));
            bmin = fminf(bmin, fminf(fabsf(lo_f(da)), fabsf(hi_f(da))));
            const unsigned m0 = __ballot_sync(0xffffffffu, lo_f(da) < 0.0f);
            const unsigned m1 = __ballot_sync(0xffffffffu, hi_f(da) < 0.0f);
            if (lane == 0) S.mask[q][0] = ((unsigned long long)m1 << 32) | m0;
        }
    }
    const bool band = S.u.force != 0 || bmin <= 1.0f;
    __syncwarp();
    long long exact = 0;
    if constexpr (!kDensity) {
        // few banded candidate lanes (the common case): those lanes' candidates
        // against the queries; else (or force) every query against the block
        const unsigned fl = __ballot_sync(0xffffffffu, band);
        if (fl) {
            if (S.u.force == 0 && __popc(fl) <= kBandLanes) resolve_band_lanes<kSym>(S, a, lane, b0, n, fl, exact);
            else resolve_band<kSym>(S, a, lane, b0, n, exact);
        }
    }
    // self is never its own neighbor (R12); counts; the final masks recorded
    // for the fill pass (chunk kk = us0 / 64 + k of the unit) straight from
    // the lanes that own the queries
    int inc[2] = {0, 0};
    int nzw = 0;  // non-zero mask words of this lane's queries
    unsigned long long *const dst =
        (!kDensity && S.u.rec_ok) ? a.masks + S.u.mask_base + (long long)(us0 >> 6) * nq : nullptr;
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int q = lane + 32 * h;
        if (q < nq) {
            const int sl = S.self[q] - us0;
            unsigned long long m0 = S.mask[q][0], m1 = nch > 1 ? S.mask[q][1] : 0ull;
            if (sl >= 0 && sl < n) {
                if (sl < 64) m0 &= ~(1ull << sl);
                else m1 &= ~(1ull << (sl - 64));
            }
            inc[h] = __popcll(m0) + __popcll(m1);
            nzw += (m0 != 0ull) + (m1 != 0ull);
            if (dst) {
                BT_DEV_CHECK(S.u.mask_base + (long long)(us0 >> 6) * nq + (nch > 1 ? nq : 0) + q < a.mask_cap);
                __stcs(&dst[q], m0);
                if (nch > 1) __stcs(&dst[nq + q], m1);
            }
        }
    }
    nzw = __reduce_add_sync(0xffffffffu, nzw);
    if (lane == 0) {
        S.u.tests += (long long)n * nq;
        S.u.exact += exact;
        S.u.nzw += nzw;
    }
    __syncwarp();
    return make_int2(inc[0], inc[1]);
}

// Flattened position p = w0 + lane of the current leaf group (w0 a multiple
// of 32) -> owning leaf (leaf starts up to p, from the group's start bitmap;
// a one-leaf group, which may be an over-full leaf, has none) and tree
// position (-1: past the end).
__device__ __forceinline__ void locate(const WalkSmem &S, int total, bool single, int w0, int lane, unsigned le,
                                       int &pos, int &mine) {
    const int w = min(w0 >> 5, kGroupPos / 32 - 1);  // (clamped: one-leaf groups ignore the bitmap)
    const int m = (int)S.lwpre[w] + __popc(S.lstart[w] & le) - 1;
    mine = single ? 0 : m;
    BT_DEV_CHECK(mine >= 0 && mine < kGroup);
    const int p = w0 + lane;
    pos = (p < total) ? p + S.ldel[mine] : -1;
}

// Stage the particles of the current leaf group from window w0 on (lemma L3
// cull) into the warp's staging buffer at nst, until the group is done or a
// whole block is staged.  kMixed: some leaf of the group is
// staged from the fp64 records (a = fl32(fl64(x - c))).
template <bool kMixed, bool kSym, bool kD>
__device__ __forceinline__ void stage_group(WalkSmemT<kD, kSym> &S, const WalkArgs &a, int lane, int total, bool single,
                                            int &w0, int &nst, int slot0) {
    const unsigned lt = lanemask_lt(), le = lt | (1u << lane);
    const float4 *__restrict__ rec32 = a.rec32;
    const float4 B0 = S.u.box0, B1 = S.u.box1;
    const int2 qn = lds2iv(&S.u.q0);
    const bool rec_ok = S.u.rec_ok != 0;
    int32_t *const cands = S.u.cand_ptr + (unsigned)slot0;
    // record of position pos: the compact record, or (large leaf of a kMixed
    // group, `rel` set) the fp64 record already relative to the unit centre
    auto load = [&](int pos, int mine, bool &rel) {
        float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
        rel = false;
        if (!kMixed) {  // past-the-end lanes read record 0 (never kept): no branch
            r = __ldg(&rec32[max(pos, 0)]);
        } else if (pos >= 0) {
            if (!kMixed || S.loff[mine].w != 0.0f) {
                r = __ldg(&rec32[pos]);
            } else {  // large leaf: exact fp64 record, a = fl32(fl64(x - c))
                const double4 d = a.rec[pos];
                r = make_float4(__double2float_rn(__dsub_rn(d.x, S.u.c[0])), __double2float_rn(__dsub_rn(d.y, S.u.c[1])),
                                __double2float_rn(__dsub_rn(d.z, S.u.c[2])), __int_as_float((int)__double_as_longlong(d.w)));
                rel = true;
            }
        }
        return r;
    };
    int pos, mine;
    bool rel;
    locate(S, total, single, w0, lane, le, pos, mine);
    float4 r = load(pos, mine, rel);
#pragma unroll 1
    for (; w0 < total; w0 += 32) {
        if (nst >= kBlk) break;  // a block is staged: the caller tests it and resumes at w0
        // the next window's record load is issued before this window is processed
        int pos_n = -1, mine_n = 0;
        bool rel_n = false;
        float4 r_n = r;
        if (w0 + 32 < total) {
            locate(S, total, single, w0 + 32, lane, le, pos_n, mine_n);
            r_n = load(pos_n, mine_n, rel_n);
        }
        // fp32 relative coordinates (compact: fl32(r32 + fl32(c_leaf - c))) and the
        // conservative fp32 Minkowski cull against the query box (L3 / L4)
        float4 of = S.loff[mine];
        if (kMixed && rel) of = make_float4(0.f, 0.f, 0.f, 0.f);
        // (x, y) as packed pairs: the same IEEE roundings as the scalar forms
        const unsigned long long axy = f2_add(pk(r.x, r.y), pk(of.x, of.y));
        const unsigned long long lxy = f2_add(axy, pk(-B0.x, -B0.y));  // a - lo (fl(lo - a) = -fl(a - lo))
        const unsigned long long hxy = f2_add(axy, pk(-B1.x, -B1.y));  // a - hi
        const float ax = lo_f(axy), ay = hi_f(axy);
        const float az = __fadd_rn(r.z, of.z);
        const float gx = fmaxf(0.0f, fmaxf(-lo_f(lxy), lo_f(hxy)));
        const float gy = fmaxf(0.0f, fmaxf(-hi_f(lxy), hi_f(hxy)));
        const float gz = fmaxf(0.0f, fmaxf(__fsub_rn(B0.z, az), __fsub_rn(az, B1.z)));
        const float g2 = __fmaf_rn(gz, gz, __fmaf_rn(gy, gy, __fmul_rn(gx, gx)));
        const bool keep = pos >= 0 && g2 < (kSym ? S.lcull[mine] : B0.w);
        const unsigned km = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const int slot = nst + __popc(km & lt);
            BT_DEV_CHECK(slot < kStg && pos >= 0 && pos < a.n_rec);
            BT_DEV_CHECK(!rec_ok || S.u.cand_base + slot0 + slot < a.cand_cap);
            S.stg[slot] = make_float4(ax, ay, az, __int_as_float(pos));
            if (rec_ok) __stcs(&cands[(unsigned)slot], a.tree_order ? pos : __float_as_int(r.w));
            if ((unsigned)(pos - qn.x) < (unsigned)qn.y) S.self[pos - qn.x] = slot0 + slot;
        }
        nst += __popc(km);
        pos = pos_n;
        mine = mine_n;
        rel = rel_n;
        r = r_n;
    }
}

#ifndef BT_WALK_MIN_BLOCKS
#define BT_WALK_MIN_BLOCKS 7
#endif
// kSym: the symmetric criterion (R22): candidates culled with their leaf's
// radius, each pair tested against both thresholds (lemma L4s)
template <bool kDensity, bool kSym>
__global__ void __launch_bounds__(kWalkThreads, BT_WALK_MIN_BLOCKS) walk_kernel(WalkArgs a) {
    __shared__ WalkSmemT<kDensity, kSym> smem[kWalkThreads / 32];
    const int lane = threadIdx.x & 31;
    WalkSmemT<kDensity, kSym> &S = smem[threadIdx.x >> 5];
    const float inf = __int_as_float(0x7f800000);
    if (lane == 0) {
        S.u.cs = Slab();
        S.u.ms = Slab();
        S.u.tests = S.u.exact = S.u.staged = S.u.loaded = S.u.nzw = 0;
    }
    __syncwarp();
    WorkBatch wb;
    unsigned long long csum = 0;  // checksum of this lane's counts (fill-only offsets validation)
    for (;;) {
        const long long uid = next_unit(wb, &a.ctr[C_WORK3], a.n_units, 1, lane);
        if (uid >= a.n_units) break;
        const UnitRun R = a.urun[uid];
        int32_t qo[2];
        int nq, q0;
        if (!kSym && !kDensity && a.uprep) {
            // the gather count pass: geometry and query records prepared by the descent
            const int4 UU = a.units[uid];
            q0 = UU.y;
            nq = UU.z;
            const UnitPrep P = a.uprep[uid];
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int k = lane + 32 * h;
                qo[h] = 0;
                if (k < nq) {
                    const float4 r = a.qrec[q0 + k];
                    qo[h] = a.tree_order ? q0 + k : a.perm[q0 + k];
                    S.q0[k] = make_float4(r.x, r.x, r.y, r.y);
                    S.q1[k] = make_float4(r.z, r.z, r.w, r.w);
                } else {  // padding query: v = Ac + 2 >= 2 (never a neighbor, never banded)
                    S.q0[k] = make_float4(0.f, 0.f, 0.f, 0.f);
                    S.q1[k] = make_float4(0.f, 0.f, 2.f, 2.f);
                }
                S.self[k] = -1;
            }
            Slab cs = S.u.cs, ms = S.u.ms;
            const long long need_c = R.loaded, need_m = (long long)((R.loaded + 63) >> 6) * nq;
            const bool okc = slab_reserve(cs, need_c, kCandSlab, a.cand_cap, &a.ctr[C_CAND], lane);
            const bool okm = slab_reserve(ms, need_m, kMaskSlab, a.mask_cap, &a.ctr[C_MASK], lane);
            __syncwarp();
            if (lane == 0) {
                S.u.cs = cs;
                S.u.ms = ms;
                S.u.cand_base = cs.cur;
                S.u.cand_ptr = a.cands + cs.cur;
                S.u.mask_base = ms.cur;
                S.u.c[0] = P.c[0];
                S.u.c[1] = P.c[1];
                S.u.c[2] = P.c[2];
                S.u.E = P.E;
                S.u.q0 = q0;
                S.u.nq = nq;
                S.u.rec_ok = okc && okm;
                S.u.force = P.k == 0.0f;
                S.u.k = P.k;
                S.u.box0 = P.box0;
                S.u.box1 = P.box1;
            }
        } else {
            UnitGeom G;
            unit_setup(a, a.units[uid], lane, G, kSym ? R.rmax : 0.0);
            nq = G.nq;
            q0 = G.q0;
            qo[0] = G.qo[0];
            qo[1] = G.qo[1];
            const double eps = l4_eps(G.E);
            float kq[2] = {INFINITY, INFINITY}, mid[2] = {0.0f, 0.0f};
            float ku;
            double tqmin = INFINITY;  // symmetric: the smallest query threshold of the unit
            if (kSym) {
#pragma unroll
                for (int h = 0; h < 2; h++)
                    if (lane + 32 * h < G.nq) {
                        tqmin = fmin(tqmin, G.qT[h]);
                        mid[h] = __double2float_rn(G.qT[h]);  // Mid_i = fl32(T_i)
                    }
                tqmin = warp_min(tqmin);
                ku = l4_band_sym(tqmin, G.Rx, G.E, eps, a.exact_only != 0);
            } else {
#pragma unroll
                for (int h = 0; h < 2; h++)
                    if (lane + 32 * h < G.nq) l4_band(G.qT[h], G.qt[h], G.E, eps, a.exact_only != 0, kq[h], mid[h]);
                // unit band scale: the minimum power of two (0 = force)
                ku = fminf(kq[0], kq[1]);
                for (int d = 16; d; d >>= 1) ku = fminf(ku, __shfl_xor_sync(0xffffffffu, ku, d));
            }
            const bool force = ku == 0.0f;
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int k = lane + 32 * h;
                if (k < G.nq) {
                    const float ax = __double2float_rn(__dsub_rn(G.qx[h], G.c[0]));
                    const float ay = __double2float_rn(__dsub_rn(G.qy[h], G.c[1]));
                    const float az = __double2float_rn(__dsub_rn(G.qz[h], G.c[2]));
                    // Q = -2 k q (exact), Bq = fl32(k (|q|^2 - Mid)), |q|^2 in fp64 from the fp32 q
                    // (symmetric: B''q = fl32(k |q|^2), -k Mid_i apart)
                    const float m2k = -2.0f * ku;
                    const double qq = (double)ax * ax + (double)ay * ay + (double)az * az;
                    const float bq = force ? 0.0f
                                           : __double2float_rn((double)ku * (qq - (kSym ? 0.0 : (double)mid[h])));
                    S.q0[k] = make_float4(m2k * ax, m2k * ax, m2k * ay, m2k * ay);
                    S.q1[k] = make_float4(m2k * az, m2k * az, bq, bq);
                    if (kSym) S.qm[k] = make_float2(-ku * mid[h], -ku * mid[h]);
                    if constexpr (kDensity) {
                        S.d.hinv[k] = (float)(1.0 / a.h_tree[G.q0 + k]);
                        S.d.qraw[k] = make_float4(ax, ay, az, 0.f);
                    }
                } else {  // padding query: v = Ac + 2 >= 2 (never a neighbor, never banded; symmetric: +inf)
                    S.q0[k] = make_float4(0.f, 0.f, 0.f, 0.f);
                    S.q1[k] = kSym ? make_float4(0.f, 0.f, inf, inf) : make_float4(0.f, 0.f, 2.f, 2.f);
                    if (kSym) S.qm[k] = make_float2(0.f, 0.f);
                }
                S.self[k] = -1;
            }
            // fp32 images of the query box and the conservative cull radius
            // (R'_u + 4 eps)(1 + 2^-20) (L3 / L4)
            float blo[3], bhi[3], cull2;
            for (int l = 0; l < 3; l++) {
                blo[l] = __double2float_rn(__dsub_rn(G.lo[l], G.c[l]));
                bhi[l] = __double2float_rn(__dsub_rn(G.hi[l], G.c[l]));
            }
            const double rc = (G.Ru + 4.0 * eps) * (1.0 + 0x1p-20);
            const double rc2 = rc * rc * (1.0 + 0x1p-40);
            cull2 = (rc2 < 3.0e38) ? __double2float_ru(rc2) : inf;
            // record space for the unit: at most `loaded` candidates
            Slab cs = S.u.cs, ms = S.u.ms;
            const long long need_c = R.loaded, need_m = (long long)((R.loaded + 63) >> 6) * G.nq;
            bool okc = false, okm = false;
            if (!kDensity) {  // the density mode records nothing
                okc = slab_reserve(cs, need_c, kCandSlab, a.cand_cap, &a.ctr[C_CAND], lane);
                okm = slab_reserve(ms, need_m, kMaskSlab, a.mask_cap, &a.ctr[C_MASK], lane);
            }
            __syncwarp();
            if (lane == 0) {
                S.u.cs = cs;
                S.u.ms = ms;
                S.u.cand_base = cs.cur;
                S.u.cand_ptr = a.cands + cs.cur;
                S.u.mask_base = ms.cur;
                S.u.c[0] = G.c[0];
                S.u.c[1] = G.c[1];
                S.u.c[2] = G.c[2];
                S.u.E = G.E;
                S.u.q0 = G.q0;
                S.u.nq = G.nq;
                S.u.rec_ok = okc && okm;
                S.u.force = force;
                S.u.k = ku;
                S.u.box0 = make_float4(blo[0], blo[1], blo[2], cull2);
                S.u.box1 = make_float4(bhi[0], bhi[1], bhi[2], 0.0f);
                if (kSym) {
                    S.u.Ru = G.Ru;
                    S.u.eps = eps;
                    S.u.tqmin = tqmin;
                }
            }
        }
        __syncwarp();
        int cnt0 = 0, cnt1 = 0;
        double dacc[2] = {0.0, 0.0};  // density mode: sum of m_j w(r_ij / h_i) of this lane's queries
        long long loaded = 0;
        const int nleaf = R.nleaf;
        const long long list_off = R.list_off;
        int nst = 0, slot0 = 0;            // candidates in the staging buffer; unit slot of stg[0]
        int g0 = 0, w0 = 0, total = 0, nl = 0;
        bool mixed = false, have_group = false;
        for (;;) {
            // ---- staging phase: stage (at least) a block
            while (g0 < nleaf) {
                if (!have_group) {
                    // the group's leaves: first position, count, offset of the centre
                    const int gi = g0 + lane;
                    int cnt = 0, beg = 0;
                    float lcull = 0.0f;
                    float4 off = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (gi < nleaf) {
                        const LeafRec *lr = a.leaf_rec + a.ulist[list_off + gi];
                        const double2 cxy = *reinterpret_cast<const double2 *>(&lr->cx);
                        const double2 czH = *reinterpret_cast<const double2 *>(&lr->cz);
                        const int2 bc = *reinterpret_cast<const int2 *>(&lr->begin);
                        beg = bc.x;
                        cnt = bc.y;
                        // leaf centre (as the build computed it) relative to the unit centre; the
                        // compact records are usable when the leaf half-extent H <= 7 E (l4_eps)
                        off = make_float4(__double2float_rn(__dsub_rn(cxy.x, S.u.c[0])),
                                          __double2float_rn(__dsub_rn(cxy.y, S.u.c[1])),
                                          __double2float_rn(__dsub_rn(czH.x, S.u.c[2])),
                                          (czH.y <= 7.0 * S.u.E) ? 1.0f : 0.0f);
                        if (kSym) {  // the leaf's cull radius: max(R'_u, R'(h_max)), fp32 image as the unit's (L3 / L4)
                            const double RL = fmax(S.u.Ru, rprime(a.leaf_hmax[a.ulist[list_off + gi]], a.M));
                            const double rc = (RL + 4.0 * S.u.eps) * (1.0 + 0x1p-20);
                            const double rc2 = rc * rc * (1.0 + 0x1p-40);
                            lcull = (rc2 < 3.0e38) ? __double2float_ru(rc2) : __int_as_float(0x7f800000);
                        }
                    }
                    int inc = cnt;
                    for (int d = 1; d < 32; d <<= 1) {
                        const int o = __shfl_up_sync(0xffffffffu, inc, d);
                        if (lane >= d) inc += o;
                    }
                    // the group: the leading leaves within kGroupPos positions (at least one)
                    nl = max(1, __popc(__ballot_sync(0xffffffffu, gi < nleaf && inc <= kGroupPos)));
                    total = __shfl_sync(0xffffffffu, inc, nl - 1);
                    S.ldel[lane] = beg - (inc - cnt);
                    S.loff[lane] = off;
                    if (kSym) S.lcull[lane] = lcull;
                    // start bitmap of the group's positions and the starts before each word
                    const int nw = nl > 1 ? (total + 31) >> 5 : 0;  // <= kGroupPos / 32
                    for (int w = lane; w < nw; w += 32) S.lstart[w] = 0u;
                    __syncwarp();
                    if (nl > 1 && lane < nl) atomicOr(&S.lstart[(inc - cnt) >> 5], 1u << ((inc - cnt) & 31));
                    __syncwarp();
                    {
                        const int c0 = lane < nw ? __popc(S.lstart[lane]) : 0;
                        const int c1 = lane + 32 < nw ? __popc(S.lstart[lane + 32]) : 0;
                        int i0 = c0, i1 = c1;
                        for (int d = 1; d < 32; d <<= 1) {
                            const int o0 = __shfl_up_sync(0xffffffffu, i0, d), o1 = __shfl_up_sync(0xffffffffu, i1, d);
                            if (lane >= d) {
                                i0 += o0;
                                i1 += o1;
                            }
                        }
                        const int t0 = __shfl_sync(0xffffffffu, i0, 31);
                        if (lane < nw) S.lwpre[lane] = (unsigned char)(i0 - c0);
                        if (lane + 32 < nw) S.lwpre[lane + 32] = (unsigned char)(t0 + i1 - c1);
                    }
                    mixed = __any_sync(0xffffffffu, lane < nl && gi < nleaf && off.w == 0.0f);
                    __syncwarp();
                    w0 = 0;
                    have_group = true;
                }
                if (mixed)
                    stage_group<true, kSym, kDensity>(S, a, lane, total, nl == 1, w0, nst, slot0);
                else
                    stage_group<false, kSym, kDensity>(S, a, lane, total, nl == 1, w0, nst, slot0);
                if (w0 < total) break;  // a block is staged
                loaded += total;
                g0 += nl;
                have_group = false;
            }
            const bool done = g0 >= nleaf;
            __syncwarp();
            // ---- test phase: the staged blocks (all but a partial last one unless done)
            const int ntest = done ? nst : nst - nst % kBlk;
            for (int b0 = 0; b0 < ntest; b0 += kBlk) {
                if constexpr (kDensity) {
                    density_block(S, a, lane, b0, min(kBlk, ntest - b0), dacc);
                    if (lane == 0) S.u.tests += (long long)min(kBlk, ntest - b0) * S.u.nq;
                } else {
                    const int2 inc = test_block<kDensity, kSym>(S, a, lane, min(kBlk, ntest - b0), slot0 + b0, b0, dacc);
                    cnt0 += inc.x;
                    cnt1 += inc.y;
                }
            }
            if (done) {
                slot0 += nst;
                break;
            }
            // move the partial block to the front of the staging buffer (rest < 32 <= ntest: no overlap)
            const int rest = nst - ntest;
            if (lane < rest) S.stg[lane] = S.stg[ntest + lane];
            slot0 += ntest;
            nst = rest;
            __syncwarp();
        }
        const int nstaged = slot0;
        if constexpr (kDensity) {
            // rho_i = (m_i w(0) + sum_j m_j w(r_ij / h_i)) / (pi h_i^3)   (R21; the dense sum holds the self term)
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int k = lane + 32 * h;
                if (k < nq) {
                    const double hi = a.h_tree[q0 + k];
                    a.rho[qo[h]] = dacc[h] / (3.14159265358979323846 * hi * hi * hi);  // (self: w(0) in the sum)
                }
            }
        } else {
            if (lane < nq) {
                a.counts[qo[0]] = cnt0;
                csum += (unsigned long long)cnt0 * (2ull * (unsigned)qo[0] + 1ull);
            }
            if (lane + 32 < nq) {
                a.counts[qo[1]] = cnt1;
                csum += (unsigned long long)cnt1 * (2ull * (unsigned)qo[1] + 1ull);
            }
        }
        __syncwarp();
        if (lane == 0) {
            UnitRun &W = a.urun[uid];
            W.cand_base = S.u.cand_base;
            W.mask_base = S.u.mask_base;
            W.nstaged = nstaged;
            W.ok = S.u.rec_ok;
            S.u.cs.cur += nstaged;
            S.u.ms.cur += (long long)((nstaged + 63) >> 6) * nq;
            S.u.staged += nstaged;
            S.u.loaded += loaded;
        }
        __syncwarp();
    }
    for (int d = 16; d; d >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, d);
    if (lane == 0) {
        if (!kDensity) atomicAdd((unsigned long long *)&a.ctr[C_CSUM], csum);
        atomicAdd((unsigned long long *)&a.ctr[C_NZW], (unsigned long long)S.u.nzw);
        atomicAdd((unsigned long long *)&a.ctr[C_TESTS], (unsigned long long)S.u.tests);
        atomicAdd((unsigned long long *)&a.ctr[C_EXACT], (unsigned long long)S.u.exact);
        atomicAdd((unsigned long long *)&a.ctr[C_STAGED], (unsigned long long)S.u.staged);
        atomicAdd((unsigned long long *)&a.ctr[C_LOADED], (unsigned long long)S.u.loaded);
    }
}

// ---------------------------------------------------------------------------
// Fill pass (A13, Alg. 2 "Add q to NeighborsOf(p)" P:294): replay the
// recorded masks into the CSR rows.  (Bounded by the DRAM cost of writing
// rows at random CSR positions: tools/probe_csr.py measured a plain
// warp-per-row writer of the same rows at 8.7 ms of this pass's 10.7 ms at
// cfg 5; POPC runs on the quarter-rate XU pipe, which
// ncu had at 71 % of its peak with four POPC per mask word -- hence the
// per-round prefix packs below; fewer ALU instructions per mask word did not
// shorten it in caller order.)  Per unit, rounds
// of up to kFillChunks (6) chunks: the chunks' candidate indices in registers (chunk k,
// lane l -> slots 64k + l, 64k + 32 + l), their masks in shared memory; for
// each (query, chunk) mask word __popc(mask & lanemask_lt) gives each
// neighbor's slot in the query's row (row order unspecified, R15).
// ---------------------------------------------------------------------------
constexpr int kFillWarps = kFillThreads / 32;
constexpr int kCsrThreads = kFillThreads;

// BT_FILL_PRE: each round's row offsets are scanned once per query (lanes =
// queries: entries before word k in the round, and the low half's popcount,
// 15 bits) so the replay loop carries no running offset and issues two POPC
// per mask word (the lane ranks) instead of four -- A/B knob
#ifndef BT_FILL_PRE
#define BT_FILL_PRE 1
#endif

struct FillSmem {
    int32_t *row[kQ];                            // next write address of each query's row
    unsigned long long mask[kFillChunks * kQ];   // the round's masks, [k][q]
#if BT_FILL_PRE
    unsigned short pre[kFillChunks * kQ];        // (entries of the round before word k) << 6 | popc(low half), [k][q]
#endif
};

// CSR row store of the fill (BT_FILL_ST: 0 streaming st.global.cs, 1 plain
// st.global, 2 st.global with an L2 evict_last policy -- A/B knob)
#ifndef BT_FILL_ST
#define BT_FILL_ST 2
#endif
__device__ __forceinline__ void row_store(int32_t *p, int32_t v, unsigned long long pol) {
#if BT_FILL_ST == 0
    __stcs(p, v);
#elif BT_FILL_ST == 1
    *p = v;
#else
    asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
#endif
}

#ifndef BT_FILL_MIN_BLOCKS
#define BT_FILL_MIN_BLOCKS 5   // 48 registers: 40 warps per SM (forced to 40 registers the replay is 18 % slower)
#endif
__global__ void __launch_bounds__(kFillThreads, BT_FILL_MIN_BLOCKS) fill_kernel(WalkArgs a) {
    __shared__ FillSmem fsm[kFillWarps];
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt(), lanebit = 1u << lane;
    FillSmem &F = fsm[threadIdx.x >> 5];
    WorkBatch wb;
    const int32_t *__restrict__ cands = a.cands;
    const unsigned long long *__restrict__ masks = a.masks;
    unsigned long long pol = 0;
#if BT_FILL_ST == 2
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#endif
    for (;;) {
        const long long u = next_unit(wb, &a.ctr[C_WORK2], a.n_units, 1, lane);
        if (u >= a.n_units) break;
        const int4 U = a.units[u];
        const UnitRun R = a.urun[u];
        const int nq = U.z;
        const int nchk = (R.nstaged + 63) >> 6;
        for (int q = lane; q < nq; q += 32)
            F.row[q] = a.nbr + a.offsets[a.tree_order ? U.y + q : a.perm[U.y + q]];
        for (int kk0 = 0; kk0 < nchk; kk0 += kFillChunks) {
            const int nk = min(kFillChunks, nchk - kk0);
            int32_t c0[kFillChunks], c1[kFillChunks];
#pragma unroll
            for (int k = 0; k < kFillChunks; k++) {
                const int s0 = 64 * (kk0 + k) + lane, s1 = s0 + 32;
                c0[k] = (k < nk && s0 < R.nstaged) ? __ldcs(&cands[R.cand_base + s0]) : -1;
                c1[k] = (k < nk && s1 < R.nstaged) ? __ldcs(&cands[R.cand_base + s1]) : -1;
            }
            __syncwarp();
            const unsigned long long *src = masks + R.mask_base + (long long)kk0 * nq;
            BT_DEV_CHECK(R.mask_base + (long long)(kk0 + nk) * nq <= a.mask_cap && R.cand_base + R.nstaged <= a.cand_cap);
            for (int w = lane; w < nk * nq; w += 32) F.mask[w] = __ldcs(&src[w]);
            __syncwarp();
#if BT_FILL_PRE
            int tot[kQ / 32];
#pragma unroll
            for (int t = 0; t < kQ / 32; t++) {
                const int q = lane + 32 * t;
                int o = 0;
                if (q < nq) {
#pragma unroll
                    for (int k = 0; k < kFillChunks; k++) {
                        if (k >= nk) break;
                        const unsigned long long m = F.mask[k * nq + q];
                        const int plo = __popc((unsigned)m);
                        F.pre[k * nq + q] = (unsigned short)((o << 6) | plo);
                        o += plo + __popc((unsigned)(m >> 32));
                    }
                }
                tot[t] = o;
            }
            __syncwarp();
            for (int q = 0; q < nq; q++) {
                int32_t *const dst = F.row[q];
#pragma unroll
                for (int k = 0; k < kFillChunks; k++) {
                    if (k >= nk) break;
                    const unsigned long long m = F.mask[k * nq + q];
                    const unsigned lo = (unsigned)m, hi = (unsigned)(m >> 32);
                    if (!(lo | hi)) continue;
                    const unsigned pk = F.pre[k * nq + q];
                    const int o = (int)(pk >> 6), plo = (int)(pk & 63u);
                    BT_DEV_CHECK(dst - a.nbr + o + plo + __popc(hi) <= a.nbr_cap);
                    if (lo & lanebit) row_store(&dst[o + __popc(lo & lt)], c0[k], pol);
                    if (hi & lanebit) row_store(&dst[o + plo + __popc(hi & lt)], c1[k], pol);
                }
            }
            __syncwarp();
#pragma unroll
            for (int t = 0; t < kQ / 32; t++)
                if (lane + 32 * t < nq) F.row[lane + 32 * t] += tot[t];
            __syncwarp();
#else
            for (int q = 0; q < nq; q++) {
                int32_t *const dst = F.row[q];
                int o = 0;  // entries of this round written to the row
#pragma unroll
                for (int k = 0; k < kFillChunks; k++) {
                    if (k >= nk) break;
                    const unsigned long long m = F.mask[k * nq + q];
                    const unsigned lo = (unsigned)m, hi = (unsigned)(m >> 32);
                    if (!(lo | hi)) continue;
                    const int plo = __popc(lo);
                    BT_DEV_CHECK(dst - a.nbr + o + plo + __popc(hi) <= a.nbr_cap);
                    if (lo & lanebit) row_store(&dst[o + __popc(lo & lt)], c0[k], pol);
                    if (hi & lanebit) row_store(&dst[o + plo + __popc(hi & lt)], c1[k], pol);
                    o += plo + __popc(hi);
                }
                if (lane == 0 && o) F.row[q] = dst + o;
            }
            __syncwarp();
#endif
        }
    }
}

// ---------------------------------------------------------------------------
// Symmetric criterion (reading R22): j is a neighbor of i
// iff d2 < (2 max(h_i, h_j))^2.  The walk finds these pairs from the query
// side: every radius of the descent, the culls and the staging becomes
// max(R'_u, R'(h_max)) with h_max the largest h of the node / leaf tested,
// and the pair test checks both thresholds (walk_kernel<.., kSym>).  These
// kernels give every leaf and internal node its h_max per search.
// ---------------------------------------------------------------------------
__global__ void leaf_hmax_kernel(const double *__restrict__ h_tree, const int32_t *__restrict__ begin,
                                 const int32_t *__restrict__ count, int64_t n_leaves, double *__restrict__ hmax) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t L = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; L < n_leaves; L += nw) {
        const int32_t b = begin[L], c = count[L];
        double m = 0.0;
        for (int32_t k = lane; k < c; k += 32) m = fmax(m, h_tree[b + k]);
        m = warp_max(m);
        if (lane == 0) hmax[L] = m;
    }
}
// internal nodes of one depth [n0, n1): every cell of the depth (one
// contiguous range of the cell table) raises its node's h_max (atomic max on
// the bit patterns: h > 0, so they order like the values); children one
// depth deeper and leaves are done
__global__ void node_hmax_kernel(const NodeRec *__restrict__ nodes, const int32_t *__restrict__ cells, int64_t n0,
                                 int64_t n1, int64_t c0, int64_t c1, const double *__restrict__ leaf_hmax,
                                 double *__restrict__ node_hmax) {
    for (int64_t g = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < c1; g += (int64_t)gridDim.x * blockDim.x) {
        const int32_t code = cells[g];
        double v = 0.0;
        if (code >= 0) v = leaf_hmax[code];
        else if (code <= -2) v = node_hmax[code_node(code)];
        if (!(v > 0.0)) continue;
        int64_t lo = n0, hi = n1 - 1;  // the node of cell g: largest i with cell_base <= g
        while (lo < hi) {
            const int64_t m = (lo + hi + 1) >> 1;
            if (nodes[m].cell_base <= g) lo = m;
            else hi = m - 1;
        }
        atomicMax((unsigned long long *)&node_hmax[lo], (unsigned long long)__double_as_longlong(v));
    }
}

// h in tree order + validation (h finite, > 0, <= 1e150) + checksum of h
// four independent gathers in flight per thread (the h loads are random 8-B reads)
__global__ void gather_h_kernel(const int32_t *__restrict__ perm, const double *__restrict__ h, int64_t n,
                                double *__restrict__ h_tree, int *bad, long long *hsum) {
    long long acc = 0;
    bool ok = true;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; k + 3 * stride < n; k += 4 * stride) {
        long long i[4];
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) i[u] = perm ? perm[k + u * stride] : k + u * stride;
#pragma unroll
        for (int u = 0; u < 4; u++) v[u] = h[i[u]];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            ok = ok && (v[u] > 0.0 && v[u] <= 1e150);
            h_tree[k + u * stride] = v[u];
            acc += __double_as_longlong(v[u]) * (2 * i[u] + 1);
        }
    }
    for (; k < n; k += stride) {
        const long long i = perm ? perm[k] : k;
        const double v = h[i];
        ok = ok && (v > 0.0 && v <= 1e150);
        h_tree[k] = v;
        acc += __double_as_longlong(v) * (2 * i + 1);
    }
    if (!ok) atomicOr(bad, 1);
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

// max over the counts and the number of rows above ngmax (out[0], out[C_OVER - C_MAXC])
__global__ void max_count_kernel(const int32_t *c, int64_t n, int64_t ngmax, long long *out) {
    int m = 0;
    unsigned over = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        m = max(m, c[i]);
        over += c[i] > ngmax;
    }
    for (int d = 16; d; d >>= 1) {
        m = max(m, __shfl_xor_sync(0xffffffffu, m, d));
        over += __shfl_xor_sync(0xffffffffu, over, d);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax((unsigned long long *)out, (unsigned long long)m);
        if (over) atomicAdd((unsigned long long *)(out + (C_OVER - C_MAXC)), (unsigned long long)over);
    }
}

// A fill-only call's offsets must be the exclusive scan of the counts of the
// recorded test pass (else rows would overlap): offsets[0] = 0, differences
// >= 0 and, when the counts are at hand (c1 [+ c2]), equal to them; the
// checksum sum_i d_i (2i + 1) mod 2^64 is compared with the walk's C_CSUM.
__global__ void check_offsets_kernel(const int64_t *__restrict__ off, int64_t n, const int32_t *__restrict__ c1,
                                     const int32_t *__restrict__ c2, long long *ctr) {
    unsigned long long s = 0;
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = off[i + 1] - off[i];
        bad = bad || d < 0 || (i == 0 && off[0] != 0);
        if (c1) bad = bad || d != (int64_t)c1[i] + (c2 ? (int64_t)c2[i] : 0);
        s += (unsigned long long)d * (2ull * (unsigned long long)i + 1ull);
    }
    for (int d = 16; d; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
    if ((threadIdx.x & 31) == 0) atomicAdd((unsigned long long *)&ctr[C_OSUM], s);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr((int *)&ctr[C_OBAD], 1);
}

thread_local int g_exact_only = 0;

}  // namespace

void set_exact_only(int on) { g_exact_only = on; }

namespace {

// masses in tree order + validation (finite, |m| <= 1e150)
__global__ void gather_m_kernel(const int32_t *__restrict__ perm, const double *__restrict__ m, int64_t n,
                                double *__restrict__ m_tree, int *bad) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const double v = m[perm ? perm[k] : k];
        if (!(fabs(v) <= 1e150)) atomicOr(bad, 1);
        m_tree[k] = v;
    }
}

struct Grids {
    unsigned d, w, f, big;
};

template <bool kDensity, bool kSym = false>
Grids walk_grids() {
    const int sms = num_sms();
    auto grid_of = [&](const void *fn, int threads) {
        int per_sm = 0;
        BT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0));
        return (unsigned)(sms * std::max(per_sm, 1));
    };
    return Grids{grid_of((const void *)desc_kernel<false, kSym>, kDescThreads),
                 grid_of((const void *)walk_kernel<kDensity, kSym>, kWalkThreads),
                 grid_of((const void *)fill_kernel, kCsrThreads), (unsigned)std::min(sms, 32)};
}

// h in tree order (validated) + its checksum
long long gather_h(TreeDev &t, const double *h, const char *who) {
    cudaStream_t st = stream();
    const int64_t n = t.n;
    DBuf<int> dbad(1);
    t.h_tree.reserve(n, 0);
    t.counters.reserve(C_N, 0);
    BT_CUDA(cudaMemsetAsync(dbad.p, 0, sizeof(int), st));
    BT_CUDA(cudaMemsetAsync(t.counters.p + C_HSUM, 0, sizeof(int64_t), st));
    {
        Phase ph("search.gather_h");
        gather_h_kernel<<<grid_for(n, 256, (int64_t)num_sms() * 16), 256, 0, st>>>(
            t.tree_order ? nullptr : t.perm.p, h, n, t.h_tree.p, dbad.p, (long long *)t.counters.p + C_HSUM);
        BT_LAUNCH("gather_h");
    }
    int hbad = 0;
    long long hsum = 0;
    read_back({{dbad.p, &hbad, sizeof(int)}, {t.counters.p + C_HSUM, &hsum, sizeof(long long)}});
    if (hbad) throw Error(BT_ERR_INPUT, std::string(who) + ": h must be finite, > 0 and <= 1e150");
    return hsum;
}

WalkArgs walk_args(TreeDev &t, const Grids &g) {
    WalkArgs a{};
    t.urun.reserve(t.n_units, 0);
    // this tree's partition (bt_set_partition): a contiguous range of the
    // Morton-ordered units; the kernels see it as units [0, n_units)
    const int64_t u0 = t.n_units * t.part / t.nparts, u1 = t.n_units * (t.part + 1) / t.nparts;
    a.rec = t.rec.p;
    a.rec32 = t.rec32.p;
    a.perm = t.perm.p;
    a.tree_order = t.tree_order ? 1 : 0;
    a.n_rec = t.n;
    a.n_cells = t.n_cells;
    a.n_leaves = t.n_leaves;
    a.cand_cap = (long long)t.arena_cands.n;
    a.mask_cap = (long long)t.arena_masks.n;
    a.h_tree = t.h_tree.p;
    a.nodes = t.nodes.p;
    a.cells = t.cells.p;
    a.leaf_begin = t.leaf_begin.p;
    a.leaf_count = t.leaf_count.p;
    a.leaf_box = t.leaf_box.p;
    a.leaf_rec = t.leaf_rec.p;
    a.units = t.units.p + u0;
    a.n_units = u1 - u0;
    a.M = t.M;
    a.root_is_leaf = t.root_is_leaf ? 1 : 0;
    a.exact_only = g_exact_only;
    a.urun = t.urun.p + u0;
    // descent batches: up to 8 units per claim while every warp still gets >= 8 claims
    a.desc_batch = (int)std::max<int64_t>(1, std::min<int64_t>(8, a.n_units / ((int64_t)g.d * (kDescThreads / 32) * 8)));
    a.ctr = (long long *)t.counters.p;
    return a;
}

void read_counters(TreeDev &t, long long *hc) { read_back({{t.counters.p, hc, C_N * sizeof(long long)}}); }
void zero_counter(TreeDev &t, int c) { BT_CUDA(cudaMemsetAsync(t.counters.p + c, 0, sizeof(int64_t), stream())); }

// Fill-only calls: the caller's offsets must be the scan of the
// recorded test pass's counts -- compared exactly when the counts are at hand
// (c1 [+ c2]) and by the checksum of the walk (C_CSUM) otherwise.
void check_offsets(TreeDev &t, const int64_t *offsets, const int32_t *c1, const int32_t *c2, bool use_sum,
                   const char *who) {
    cudaStream_t st = stream();
    zero_counter(t, C_OSUM);
    zero_counter(t, C_OBAD);
    check_offsets_kernel<<<grid_for(t.n, 256, (int64_t)num_sms() * 8), 256, 0, st>>>(offsets, t.n, c1, c2,
                                                                                     (long long *)t.counters.p);
    BT_LAUNCH("check_offsets");
    long long osum = 0, obad = 0;
    read_back({{t.counters.p + C_OSUM, &osum, sizeof(long long)}, {t.counters.p + C_OBAD, &obad, sizeof(long long)}});
    if (obad || (use_sum && osum != t.rec_csum))
        throw Error(BT_ERR_ARG, std::string(who) + ": offsets are not the exclusive scan of this tree's neighbor counts "
                                "for this h (and partition): call the count pass again");
}

// A10: candidate-leaf lists of all units; the leaf-list arena is estimated
// (grown and redone on overflow).  Leaves the counters in hc.
template <bool kSym>
void run_descent(TreeDev &t, WalkArgs &a, const Grids &g, long long *hc) {
    cudaStream_t st = stream();
    double list_per_unit = 96.0;
    const long long warps_d = (long long)g.d * (kDescThreads / 32);
    const double *h_src = a.h_src;  // fused gather of h (first pass only)
    for (int attempt = 0;; attempt++) {
        t.ulist.reserve((long long)(list_per_unit * a.n_units) + warps_d * kListSlab, 0);
        a.ulist = t.ulist.p;
        a.list_cap = (long long)t.ulist.n;
        a.h_src = h_src;
        for (int c : {C_WORK, C_LIST, C_BIG, C_WORK4, C_NEEDC, C_NEEDM}) zero_counter(t, c);
        if (h_src) {
            zero_counter(t, C_HSUM);
            zero_counter(t, C_HBAD);
        }
        {
            Phase ph("search.desc");
            desc_kernel<false, kSym><<<g.d, kDescThreads, 0, st>>>(a);
            BT_LAUNCH("walk_desc");
        }
        read_counters(t, hc);
        if (h_src && hc[C_HBAD]) return;  // invalid h: the caller reports it (no arena growth for r = inf)
        t.big_units = hc[C_BIG];
        if (hc[C_BIG] > 0 && hc[C_LIST] <= a.list_cap) {
            // units beyond the shared-memory frontier / list reserve
            t.front.reserve((long long)g.big * (kDescThreads / 32) * 2 * std::max<int64_t>(t.n_nodes, 1), 0);
            a.front = t.front.p;
            a.front_cap = std::max<int64_t>(t.n_nodes, 1);
            a.h_src = nullptr;  // (h_tree is complete after the first pass)
            Phase ph("search.desc_big");
            desc_kernel<true, kSym><<<g.big, kDescThreads, 0, st>>>(a);
            BT_LAUNCH("walk_desc_big");
            read_counters(t, hc);
        }
        if (hc[C_LIST] <= a.list_cap) break;
        list_per_unit = 1.25 * (double)hc[C_LIST] / (double)std::max<int64_t>(1, a.n_units);
        if (attempt > 2) throw Error(BT_ERR_OOM, "bt_find_neighbors: leaf-list arena does not converge");
    }
    t.list_entries = hc[C_LIST];
    a.h_src = nullptr;
}

}  // namespace

namespace {

// h_max of every leaf and internal node (symmetric criterion): leaves from
// h_tree, internal nodes bottom-up, one launch per depth
void compute_hmax(TreeDev &t) {
    cudaStream_t st = stream();
    const int sms = num_sms();
    t.leaf_hmax.reserve(std::max<int64_t>(t.n_leaves, 1), 0);
    t.node_hmax.reserve(std::max<int64_t>(t.n_nodes, 1), 0);
    leaf_hmax_kernel<<<grid_for(t.n_leaves * 32, 256, (int64_t)sms * 16), 256, 0, st>>>(
        t.h_tree.p, t.leaf_begin.p, t.leaf_count.p, t.n_leaves, t.leaf_hmax.p);
    BT_LAUNCH("leaf_hmax");
    if (t.n_nodes > 0) BT_CUDA(cudaMemsetAsync(t.node_hmax.p, 0, t.n_nodes * sizeof(double), st));
    for (int64_t d = (int64_t)t.level_begin.size() - 2; d >= 0; d--) {
        const int64_t n0 = t.level_begin[d], n1 = t.level_begin[d + 1];
        if (n1 <= n0) continue;
        const int64_t c0 = t.level_cells[d], c1 = t.level_cells[d + 1];
        node_hmax_kernel<<<grid_for(c1 - c0, 256, (int64_t)sms * 16), 256, 0, st>>>(
            t.nodes.p, t.cells.p, n0, n1, c0, c1, t.leaf_hmax.p, t.node_hmax.p);
        BT_LAUNCH("node_hmax");
    }
}

template <bool kSym>
void search(TreeDev &t, const double *h, int32_t *counts, int64_t *offsets, int32_t *nbr_idx, int64_t capacity,
            bool count_pass, bool fill_pass) {
    cudaStream_t st = stream();
    const int64_t n = t.n;
    const char *who = kSym ? "bt_find_neighbors_sym" : "bt_find_neighbors";
    if (n == 0) {
        if (offsets && count_pass) BT_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int64_t), st));
        t.total_pairs = t.max_count = t.staged = t.loaded = t.tests = t.exact_tests = t.rows_over_ngmax = 0;
        BT_CUDA(cudaStreamSynchronize(st));
        return;
    }
    const int sms = num_sms();
    // the gather walk of a count call gathers h in its descent (each unit's
    // queries; validation and checksum as gather_h_kernel's); fill-only calls
    // (the record check needs the checksum first), partitioned trees and the
    // symmetric walk (its staging reads every candidate's h) gather first
    const bool fuse = !kSym && count_pass && t.nparts == 1;
    long long hsum = 0;
    if (fuse) {
        t.h_tree.reserve(n, 0);
        t.counters.reserve(C_N, 0);
    } else {
        hsum = gather_h(t, h, who);
    }
    const Grids g = walk_grids<false, kSym>();

    // the recorded masks of a previous test pass are reused by a fill-only
    // call when the tree, h pointer, exactness mode, criterion and h checksum all match
    const bool have_record = t.rec_valid && t.rec_h == h && t.rec_hsum == hsum && t.rec_exact == g_exact_only &&
                             t.rec_sym == kSym && t.rec_tree_order == t.tree_order;
    const bool run_test = count_pass || !have_record;

    WalkArgs a = walk_args(t, g);
    a.offsets = offsets;
    a.nbr = nbr_idx;
    a.nbr_cap = capacity;
    auto zero = [&](int c) { zero_counter(t, c); };

    DBuf<int32_t> tmp_counts;
    const int32_t *cnt_now = nullptr;  // counts of a test pass run by this call
    if (run_test) {
        int32_t *cnt = counts;
        if (!cnt) {
            tmp_counts.alloc(n);
            cnt = tmp_counts.p;
        }
        // partitioned tree: particles of other parts keep count 0 (empty rows)
        if (t.nparts > 1) BT_CUDA(cudaMemsetAsync(cnt, 0, n * sizeof(int32_t), st));
        a.counts = cnt;
        if (kSym) {
            Phase ph("search.hmax");
            compute_hmax(t);
            a.leaf_hmax = t.leaf_hmax.p;
            a.node_hmax = t.node_hmax.p;
        }
        long long hc[C_N];
        t.rec_valid = false;
        if (fuse) {
            a.h_src = h;
            a.h_out = t.h_tree.p;
        }
        if (!kSym) {  // the descent prepares the gather walk's unit geometry and query records
            const int64_t u0 = t.n_units * t.part / t.nparts;
            t.uprep.reserve(t.n_units, 0);
            t.qrec.reserve(n, 0);
            a.uprep = t.uprep.p + u0;
            a.qrec = t.qrec.p;
        }
        run_descent<kSym>(t, a, g, hc);
        if (fuse) {
            if (hc[C_HBAD]) throw Error(BT_ERR_INPUT, std::string(who) + ": h must be finite, > 0 and <= 1e150");
            hsum = hc[C_HSUM];
        }
        const long long warps_w = (long long)g.w * (kWalkThreads / 32);
        {  // A10 staging + A11 pair tests, counts, masks; candidate and mask arenas: exact bounds from the descent
            t.arena_cands.reserve(hc[C_NEEDC] + warps_w * kCandSlab, 0);
            t.arena_masks.reserve(hc[C_NEEDM] + warps_w * kMaskSlab, 0);
            a.cands = t.arena_cands.p;
            a.cand_cap = (long long)t.arena_cands.n;
            a.masks = t.arena_masks.p;
            a.mask_cap = (long long)t.arena_masks.n;
            for (int c : {C_WORK3, C_CAND, C_MASK, C_STAGED, C_LOADED, C_TESTS, C_EXACT, C_CSUM, C_NZW}) zero(c);
            {
                Phase ph("search.count");
                walk_kernel<false, kSym><<<g.w, kWalkThreads, 0, st>>>(a);
                BT_LAUNCH(kSym ? "walk_test_sym" : "walk_test");
            }
            // (the walk's counters are read with the offsets total below: one host read)
        }
        cnt_now = cnt;
        if (count_pass) {
            DBuf<long long> dtot(1);
            Phase ph("search.scan");
            device_scan<long long>(CountIn{cnt}, OffsetOut{offsets}, n, dtot.p);
            write_total_kernel<<<1, 1, 0, st>>>(offsets, n, dtot.p);
            BT_LAUNCH("write_total");
            zero(C_MAXC);
            zero(C_OVER);
            max_count_kernel<<<grid_for(n, 256, (int64_t)sms * 8), 256, 0, st>>>(cnt, n, t.ngmax,
                                                                                  (long long *)t.counters.p + C_MAXC);
            BT_LAUNCH("max_count");
        }
    }
    int64_t total = 0;
    long long hw[C_N];
    read_back({{offsets + n, &total, sizeof(int64_t)}, {t.counters.p, hw, C_N * sizeof(long long)}});
    if (run_test) {
        const bool fits = hw[C_CAND] <= (long long)t.arena_cands.n && hw[C_MASK] <= (long long)t.arena_masks.n;
        if (!fits) throw Error(BT_ERR_CUDA, std::string(who) + ": internal: walk arena bound exceeded");
        t.rec_valid = true;
        t.rec_csum = hw[C_CSUM];
        t.rec_h = h;
        t.rec_hsum = hsum;
        t.rec_exact = g_exact_only;
        t.rec_sym = kSym;
        t.rec_tree_order = t.tree_order;
        t.staged = hw[C_STAGED];
        t.loaded = hw[C_LOADED];
        t.tests = hw[C_TESTS];
        t.exact_tests = hw[C_EXACT];
        t.mask_words = hw[C_MASK];
        t.cand_slots = hw[C_CAND];
        t.mask_words_nz = hw[C_NZW];
    }
    if (count_pass) {
        t.max_count = hw[C_MAXC];
        t.rows_over_ngmax = hw[C_OVER];
    }
    t.total_pairs = total;
    if (!fill_pass || nbr_idx == nullptr) return;
    if (total > capacity)
        throw Error(BT_ERR_CAPACITY, std::string(who) + ": " + std::to_string(total) + " neighbor pairs exceed capacity " +
                                         std::to_string(capacity));
    if (!t.rec_valid) throw Error(BT_ERR_CUDA, std::string(who) + ": internal: no recorded test pass");
    if (!count_pass) check_offsets(t, offsets, cnt_now, nullptr, true, kSym ? "bt_fill_neighbors_sym" : "bt_fill_neighbors");
    a.masks = t.arena_masks.p;
    a.cands = t.arena_cands.p;
    zero(C_WORK2);
    {
        Phase ph("search.fill");
        fill_kernel<<<g.f, kCsrThreads, 0, st>>>(a);
        BT_LAUNCH("walk_fill");
    }
    BT_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

void find_neighbors(TreeDev &t, const double *h, int32_t *counts, int64_t *offsets, int32_t *nbr_idx,
                    int64_t capacity, bool count_pass, bool fill_pass, bool sym) {
    if (sym) search<true>(t, h, counts, offsets, nbr_idx, capacity, count_pass, fill_pass);
    else search<false>(t, h, counts, offsets, nbr_idx, capacity, count_pass, fill_pass);
}

// SPH density with the neighbor search fused in: the
// descent and the walk as in find_neighbors, the walk in density mode (no
// masks, no candidate records, no CSR); rho in caller order.
void density(TreeDev &t, const double *h, const double *mass, double *rho) {
    cudaStream_t st = stream();
    const int64_t n = t.n;
    if (n == 0) {
        BT_CUDA(cudaStreamSynchronize(st));
        return;
    }
    gather_h(t, h, "bt_density");
    {
        DBuf<int> dbad(1);
        BT_CUDA(cudaMemsetAsync(dbad.p, 0, sizeof(int), st));
        t.m_tree.reserve(n, 0);
        gather_m_kernel<<<grid_for(n, 256, (int64_t)num_sms() * 16), 256, 0, st>>>(t.tree_order ? nullptr : t.perm.p, mass,
                                                                                  n, t.m_tree.p, dbad.p);
        BT_LAUNCH("gather_m");
        int mbad = 0;
        read_back({{dbad.p, &mbad, sizeof(int)}});
        if (mbad) throw Error(BT_ERR_INPUT, "bt_density: masses must be finite and |m| <= 1e150");
    }
    const Grids g = walk_grids<true>();
    WalkArgs a = walk_args(t, g);
    a.m_tree = t.m_tree.p;
    a.rho = rho;
    long long hc[C_N];
    t.rec_valid = false;  // the density walk records no masks
    run_descent<false>(t, a, g, hc);
    for (int c : {C_WORK3, C_CAND, C_MASK, C_STAGED, C_LOADED, C_TESTS, C_EXACT, C_CSUM, C_NZW}) zero_counter(t, c);
    {
        Phase ph("density.walk");
        walk_kernel<true, false><<<g.w, kWalkThreads, 0, st>>>(a);
        BT_LAUNCH("walk_density");
    }
    read_counters(t, hc);
    t.staged = hc[C_STAGED];
    t.loaded = hc[C_LOADED];
    t.tests = hc[C_TESTS];
    t.exact_tests = hc[C_EXACT];
}

}  // namespace bt
