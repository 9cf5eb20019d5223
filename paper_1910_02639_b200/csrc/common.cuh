// common.cuh -- shared device/host definitions of the CUDA b-tree library.
// Citations: P:n = PAPER.md line n (arXiv 1910.02639); R-numbers = readings in
// DESIGN.md section 3.  Nothing here is shared with oracle/ (independent code).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include <stdexcept>
#include <string>
#include <initializer_list>
#include <vector>

#include "../../include/btree.h"

namespace bt {

// ---------------------------------------------------------------------------
// Errors: thrown inside the library, converted to bt_status at the ABI.
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return;
    int code = (e == cudaErrorMemoryAllocation) ? BT_ERR_OOM : BT_ERR_CUDA;
    cudaGetLastError();  // clear sticky-free errors
    throw Error(code, std::string(what) + ": " + cudaGetErrorString(e));
}
#define BT_CUDA(x) ::bt::cuda_check((x), #x)
#define BT_LAUNCH(name) ::bt::after_launch(name)

cudaStream_t stream();  // this thread's stream
void after_launch(const char *name);

// Phase profiling (CUDA events on the library stream).
struct Phase {
    const char *name;
    bool on;
    cudaEvent_t a, b;
    explicit Phase(const char *n);
    ~Phase();
};

// Device allocation through the per-thread block cache (abi.cu).
void *dmalloc(size_t bytes);
void dfree(void *p);

template <class T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf &operator=(DBuf &&o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        p = count ? static_cast<T *>(dmalloc(count * sizeof(T))) : nullptr;
    }
    // grow (preserving the first `keep` elements) to at least `count`
    void reserve(size_t count, size_t keep) {
        if (count <= n) return;
        size_t cap = count + count / 2 + 1024;
        T *q = static_cast<T *>(dmalloc(cap * sizeof(T)));
        if (keep && p) BT_CUDA(cudaMemcpyAsync(q, p, keep * sizeof(T), cudaMemcpyDeviceToDevice, stream()));
        release();
        p = q;
        n = cap;
    }
    void release() {
        if (p) dfree(p);
        p = nullptr;
        n = 0;
    }
};

// Pinned host scratch for the few control scalars read back per level.
struct HostScratch {
    int64_t *p = nullptr;
    HostScratch() { BT_CUDA(cudaMallocHost(&p, 64 * sizeof(int64_t))); }
    ~HostScratch() { if (p) cudaFreeHost(p); }
};
HostScratch &host_scratch();

// Device -> host control reads through pinned scratch (pageable destinations
// would make every small copy a staged, synchronous transfer); syncs the stream.
struct ReadBack {
    const void *src;
    void *dst;
    size_t bytes;
};
void read_back(std::initializer_list<ReadBack> items);

// ---------------------------------------------------------------------------
// Tree representation in HBM.
// ---------------------------------------------------------------------------
struct NodeRec {      // one internal node
    double lo[3];     // x_{l,min}
    double ext[3];    // x_{l,max} - x_{l,min}  (Eq. 2 denominator)
    int32_t b;        // accepted branching factor per dimension
    int32_t depth;
    int64_t cell_base;  // first entry of this node's b^3 cells in the cell table
    double bx[3];     // fl(b_l / ext): cell_coord_fast's multiplier (set with b)
    int32_t bz;       // sub-cells along z: b, or 1 for the k = 2 policies (R23)
    int32_t pad_;
};

// cell table code: -1 empty, >= 0 leaf id, <= -2 internal node (id = -2 - code)
__host__ __device__ inline int32_t node_code(int32_t node) { return -2 - node; }
__host__ __device__ inline int32_t code_node(int32_t code) { return -2 - code; }

struct LeafRec {             // per leaf, what a walk staging group reads (one 48-B record)
    double cx, cy;          // leaf centre 0.5 (lo + hi) per axis (the compact records' origin)
    double cz, H;           // ... and half-extent 0.5 max_l (hi_l - lo_l)
    int32_t begin, count;   // first tree position, particles
    int32_t pad_[2];
};

struct UnitRun {             // per walk unit, written by the walk kernels
    long long list_off;     // first candidate leaf of the unit in the leaf-list arena
    long long cand_base;    // first candidate slot of the unit (caller indices, for the fill)
    long long mask_base;    // mask word (chunk kk, query q) at mask_base + kk * nq + q
    int nleaf;              // candidate leaves (-1: descent overflowed, redo in the big pass)
    int loaded;             // particle records of the candidate leaves (arena bound)
    int nstaged;            // candidates kept by the per-particle cull
    int ok;                 // the unit's masks and candidate indices were recorded
    double rmax;            // symmetric criterion: largest cull radius max(R'_u, R'(h_max of a kept leaf))
};

struct UnitPrep {            // gather walk: a unit's geometry, prepared by the descent (A10)
    double c[3], E;         // unit centre, coordinate bound (L4)
    float4 box0, box1;      // fp32 query box relative to c: (lo xyz, cull2), (hi xyz, -)
    float k;                // band scale (power of two; 0: force)
    int pad;
};

struct TreeDev {
    int64_t n = 0;
    int32_t s = 64;
    double beta = 0.5, alpha = 0.5;
    int32_t depth_cap = 64;
    bool octree = false;       // FixedOctree / quadtree policy: b = 2 at every node, no ratio test
    int32_t dims = 3;          // k: 3, or 2 (x, y subdivided, z one slab; R23)
    // records in tree (depth-first leaf) order: x, y, z, caller index (bits)
    DBuf<double4> rec;
    // compact records in tree order: fl32(fl64(x - c_leaf)) per axis, caller index (int bits)
    DBuf<float4> rec32;
    DBuf<int32_t> perm;        // caller index of each tree position (as rec / rec32 .w)
    DBuf<NodeRec> nodes;       // internal nodes, all levels
    int64_t n_nodes = 0;
    std::vector<int64_t> level_begin;  // node ids of depth d: [level_begin[d], level_begin[d + 1])
    std::vector<int64_t> level_cells;  // their cells: [level_cells[d], level_cells[d + 1]) of the cell table
    DBuf<int32_t> cells;       // cell table, all levels
    int64_t n_cells = 0;
    DBuf<int32_t> leaf_begin;  // tree-order position of each leaf (depth-first order)
    DBuf<int32_t> leaf_count;
    DBuf<int32_t> leaf_depth;
    DBuf<double> leaf_box;     // [6*L]: lo x,y,z, hi x,y,z (tight, exact min/max)
    DBuf<LeafRec> leaf_rec;    // [L]: centre, half-extent, begin, count (walk staging)
    int64_t n_leaves = 0;
    DBuf<int32_t> leaf_id_of_level;  // scratch
    DBuf<int4> units;          // {leaf, first query (tree pos), n queries, 0}
    int64_t n_units = 0;
    int32_t part = 0, nparts = 1;  // bt_set_partition: searches cover units [n_units part / nparts, n_units (part+1) / nparts)
    double box_lo[3] = {0, 0, 0}, box_hi[3] = {0, 0, 0};
    double M = 0.0;            // max |root box coordinate|
    int32_t depth = 0, root_b = 0;
    int64_t halvings = 0, overfull = 0, max_leaf = 0;
    bool root_is_leaf = true;
    // search scratch
    DBuf<double> h_tree;       // h in tree order
    DBuf<double> leaf_hmax, node_hmax;  // symmetric criterion: max h per leaf / per node subtree
    DBuf<double> m_tree;       // masses in tree order (density consumer)
    DBuf<UnitRun> urun;                    // per-unit walk record
    DBuf<UnitPrep> uprep;                  // gather walk: per-unit geometry from the descent
    DBuf<float4> qrec;                     // gather walk: per-query record (-2k q, fl32(k(|q|^2 - Mid))) by tree position
    DBuf<int32_t> ulist;                   // candidate leaf lists of all units
    DBuf<unsigned long long> arena_masks;  // neighbor masks per (64-candidate chunk, query)
    DBuf<int32_t> arena_cands;             // candidate caller indices per slot
    bool rec_valid = false;    // arena holds the test pass of (rec_h, rec_hsum, rec_exact)
    const double *rec_h = nullptr;
    long long rec_hsum = 0;
    long long rec_csum = 0;    // checksum of the recorded pass's counts (fill-only offsets validation)
    int rec_exact = 0;
    bool rec_sym = false;      // the recorded pass is the symmetric criterion's
    bool rec_tree_order = false;  // ... and in the tree-order index space
    bool tree_order = false;   // bt_set_tree_order: h, mass, counts, offsets, rho and neighbor indices by tree position
    DBuf<int64_t> counters;    // [8] device counters (staged, tests, exact, max_count, ...)
    DBuf<int32_t> front;       // descent frontier scratch of the big-unit pass (per warp)

    int64_t total_pairs = 0, max_count = 0, staged = 0, loaded = 0, tests = 0, exact_tests = 0;
    int64_t ngmax = 512, rows_over_ngmax = 0;  // the last count's ngmax and its rows above it
    int64_t mask_words = 0, cand_slots = 0, list_entries = 0, big_units = 0, mask_words_nz = 0;
};

// Build (build.cu) and search (walk.cu) entry points.
void build_tree(TreeDev &t, const double *pos);
// sym: the symmetric max(h_i, h_j) criterion (R22) instead of the gather one
void find_neighbors(TreeDev &t, const double *h, int32_t *counts, int64_t *offsets,
                    int32_t *nbr_idx, int64_t capacity, bool count_pass, bool fill_pass, bool sym = false);

void density(TreeDev &t, const double *h, const double *mass, double *rho);

void set_exact_only(int on);
int release_cache();

// ---------------------------------------------------------------------------
// Eq. 2 with the clamp of reading R8, evaluated exactly as
//   floor( ((x - lo) / ext) * b ),  ext = x_max - x_min,
// one IEEE rounding per operation (no contraction: explicit _rn intrinsics).
// Build and walk call this same function with the same stored (lo, ext, b)
// of a node, which makes the walk's Eq. 5 ranges consistent with the build's
// distribution (lemma L2).  NaN (0/0 on a zero-extent box) -> 0.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int cell_coord(double x, double lo, double ext, int b) {
    double q = __dmul_rn(__ddiv_rn(__dsub_rn(x, lo), ext), (double)b);
    double f = floor(q);
    if (!(f >= 0.0)) return 0;
    if (f > (double)(b - 1)) return b - 1;
    return (int)f;
}

// cell_coord without the division in the common case: q = fl(fl(x - lo) *
// fl(b / ext)) differs from Eq. 2's fl(fl(fl(x - lo) / ext) * b) by at most a
// few ulps of q (|q - q_eq2| <= |q| 2^-50.9), so the two floors agree unless q
// lies within |q| 2^-45 of an integer; there (and for non-finite q) the exact
// Eq. 2 evaluation decides.  Results are identical to cell_coord's.
__device__ __forceinline__ int cell_coord_fast(double x, double lo, double ext, double bx, int b) {
    const double q = __dmul_rn(__dsub_rn(x, lo), bx);
    const double f = floor(q);
    const double m = fabs(q) * 0x1p-45 + 0x1p-1000;
    if (__dsub_rn(q, f) > m && __dsub_rn(__dadd_rn(f, 1.0), q) > m) {  // false for NaN / inf
        if (!(f >= 0.0)) return 0;
        if (f > (double)(b - 1)) return b - 1;
        return (int)f;
    }
    return cell_coord(x, lo, ext, b);
}

// Device-side bounds checks of the checked build (nvcc -DBT_CHECKED,
// tools/gpu_checked.sh): a failed check prints its location and traps, which
// surfaces as a CUDA error at the ABI.  Compiled out otherwise.
#ifdef BT_CHECKED
#define BT_DEV_CHECK(c)                                                                 \
    do {                                                                                \
        if (!(c)) {                                                                     \
            printf("BT_DEV_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);          \
            __trap();                                                                   \
        }                                                                               \
    } while (0)
#else
#define BT_DEV_CHECK(c) \
    do {                \
    } while (0)
#endif

constexpr int kWarp = 32;

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

int num_sms();  // SM count of the current device (abi.cu; cached per device)

inline unsigned grid_for(int64_t n, int threads, int64_t max_blocks = 1 << 20) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > max_blocks) b = max_blocks;
    return (unsigned)b;
}

}  // namespace bt
