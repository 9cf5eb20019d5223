// build.cu -- BuildTree (Alg. 1) as level-synchronous device kernels.
//
// All nodes of one depth are processed together ("level").  For a level:
//   A2  Eq. 1 per node: b0 = smallest b >= 2 with b^3 s >= n_i   (level_b)
//   A3  Eq. 2 + Eq. 3 key per active particle, A4 histogram       (key_hist)
//   A5  Eq. 4 ratio, halve b while r >= beta and b > 2; redo A3/A4 for the
//       halved nodes only                                         (under_count, ratio_decide)
//   A6  one scan over the level's cells -> in-node offsets, child node ids,
//       next-level positions, leaf ids                            (device_scan)
//   A8  emit child nodes (equal 1/b slices of the parent box), leaves and the
//       cell table                                                (emit)
//   A7  counting-sort scatter of the particle records: leaf cells go to their
//       final tree-order position, child-node cells to the next level's
//       active array                                              (scatter)
// After the last level: A9 per leaf, sort by caller index (canonical order,
// SPEC S:180), tight bounding box; work units of <= 64 queries.
//
// The tree order is the paper's depth-first walk order (Sec. IV-E):
// a node's particles occupy one contiguous range, its sub-cells follow in
// ascending j, recursively.
#include <algorithm>
#include <cmath>
#include <cstring>

#include <cub/device/device_segmented_sort.cuh>

#include "common.cuh"
#include "scan.cuh"

namespace bt {

namespace {

constexpr int kThreads = 256;
// BT_RANK_HIST: the histogram's atomic returns each particle's rank in its
// cell and the scatter adds it to the cell's start (one atomic per particle
// and round instead of one in the histogram and one in the scatter) -- A/B knob
#ifndef BT_RANK_HIST
#define BT_RANK_HIST 0
#endif
#ifndef BT_SCATTER_UNROLL
#define BT_SCATTER_UNROLL 4  // particles per thread in flight in key_hist / scatter
#endif

struct LevelNode {
    int32_t act_begin;   // first active particle of this node (level array)
    int32_t count;       // n_i
    int32_t final_begin; // first tree-order position of the node's range
    int32_t gid;         // global node id (NodeRec index)
    int32_t b0;          // Eq. 1
    int32_t b;           // current / accepted branching factor
    int32_t flag;        // (re)distribute in this round
    int32_t halvings;
    int32_t kz;          // 1: z is divided like x, y (k = 3); 0: one z slab (k = 2, R23)
    int32_t pad_;
    int64_t cell_base;   // level-local first cell
    int64_t under;       // #{j < b^3 : n_j <= alpha s}   (Eq. 4 numerator)
    double bx[3];        // fl(b / ext) of the current b (cell_coord_fast)
};

struct CellScan {  // per-cell values scanned in one pass (A6)
    long long pre;     // particles before this cell (level-wide)
    long long actoff;  // particles of child-node cells before this cell
    long long ncnext;  // sub-cells (Eq. 1 b0^k) of the child nodes before this cell: the next level's cell count
    int nnode;         // child-node cells before this cell
    int nleaf;         // leaf cells before this cell
    int maxleaf;       // largest leaf cell (max, not sum: the combine is still associative)
    int pad_;
    __host__ __device__ CellScan operator+(const CellScan &o) const {
        return CellScan{pre + o.pre, actoff + o.actoff, ncnext + o.ncnext, nnode + o.nnode, nleaf + o.nleaf,
                        maxleaf > o.maxleaf ? maxleaf : o.maxleaf, 0};
    }
};

// ---- A1: records + bounding box -------------------------------------------
__global__ void __launch_bounds__(kThreads) pack_bbox_kernel(const double *__restrict__ pos, int64_t n,
                                                             double4 *__restrict__ rec, double *partials,
                                                             int *bad) {
    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    int badv = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double x = pos[3 * i], y = pos[3 * i + 1], z = pos[3 * i + 2];
        // finite and |x| <= 1e150 (keeps squared distances finite)
        if (!(fabs(x) <= 1e150) || !(fabs(y) <= 1e150) || !(fabs(z) <= 1e150)) badv = 1;
        if (rec) rec[i] = make_double4(x, y, z, __longlong_as_double((long long)i));
        mn[0] = fmin(mn[0], x); mn[1] = fmin(mn[1], y); mn[2] = fmin(mn[2], z);
        mx[0] = fmax(mx[0], x); mx[1] = fmax(mx[1], y); mx[2] = fmax(mx[2], z);
    }
    if (badv) atomicOr(bad, 1);
    __shared__ double sh[6][kThreads / 32];
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int l = 0; l < 3; l++) {
        double a = mn[l], b = mx[l];
        for (int d = 16; d; d >>= 1) {
            a = fmin(a, __shfl_xor_sync(0xffffffffu, a, d));
            b = fmax(b, __shfl_xor_sync(0xffffffffu, b, d));
        }
        if (lane == 0) { sh[l][wid] = a; sh[3 + l][wid] = b; }
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        int l = threadIdx.x;
        double a = INFINITY, b = -INFINITY;
        for (int w = 0; w < kThreads / 32; w++) { a = fmin(a, sh[l][w]); b = fmax(b, sh[3 + l][w]); }
        partials[6 * blockIdx.x + l] = a;
        partials[6 * blockIdx.x + 3 + l] = b;
    }
}

// Root box: exact min/max, each side expanded by max(1e-9 * extent, 1e-12)
// (reading R9).  Writes the root NodeRec lo/ext and box[0..6], M.
__global__ void __launch_bounds__(256) root_box_kernel(const double *partials, int nblocks, NodeRec *root,
                                                       double *box) {
    __shared__ double sh[6][8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double v[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    for (int k = threadIdx.x; k < nblocks; k += blockDim.x)
        for (int l = 0; l < 3; l++) {
            v[l] = fmin(v[l], partials[6 * k + l]);
            v[3 + l] = fmax(v[3 + l], partials[6 * k + 3 + l]);
        }
    for (int l = 0; l < 6; l++) {
        for (int d = 16; d; d >>= 1) {
            double o = __shfl_xor_sync(0xffffffffu, v[l], d);
            v[l] = l < 3 ? fmin(v[l], o) : fmax(v[l], o);
        }
        if (lane == 0) sh[l][wid] = v[l];
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    double M = 0.0;
    for (int l = 0; l < 3; l++) {
        double a = INFINITY, b = -INFINITY;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) { a = fmin(a, sh[l][w]); b = fmax(b, sh[3 + l][w]); }
        double pad = __dmul_rn(1e-9, __dsub_rn(b, a));
        if (pad < 1e-12) pad = 1e-12;
        double lo = __dsub_rn(a, pad), hi = __dadd_rn(b, pad);
        box[l] = lo;
        box[3 + l] = hi;
        root->lo[l] = lo;
        root->ext[l] = __dsub_rn(hi, lo);
        M = fmax(M, fmax(fabs(lo), fabs(hi)));
    }
    box[6] = M;
    root->depth = 0;
    root->b = 0;
    root->cell_base = 0;
}

// ---- A2: Eq. 1 --------------------------------------------------------------
__host__ __device__ __forceinline__ int64_t ipow_k(int64_t b, int k) { return k == 3 ? b * b * b : b * b; }

// smallest integer b >= 2 with b^k s >= n (R6; k = 2: R23)
__host__ __device__ __forceinline__ int eq1_branching(int64_t n, int64_t s, int k) {
    int64_t m = (n + s - 1) / s;  // b^k s >= n  <=>  b^k >= ceil(n/s)
    int64_t b = (int64_t)(k == 3 ? cbrt((double)m) : sqrt((double)m));
    if (b < 2) b = 2;
    while (b > 2 && ipow_k(b - 1, k) >= m) b--;
    while (ipow_k(b, k) < m) b++;
    return (int)b;
}

// sub-cells along z: b (k = 3) or 1 (k = 2: the z axis is one slab)
__host__ __device__ __forceinline__ int bz_of(int b, int kz) { return kz ? b : 1; }

// sub-cells of a node of `count` particles (Eq. 1 b0, before any halving)
__host__ __device__ __forceinline__ long long node_cells(int64_t count, int64_t s, int octree, int dims) {
    const int b = octree ? 2 : eq1_branching(count, s, dims);
    return (long long)b * b * bz_of(b, dims == 3 ? 1 : 0);
}

__global__ void level_b_kernel(LevelNode *ln, int64_t nn, int64_t s, int octree, int dims, const NodeRec *nodes) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nn) return;
    // FixedOctree / quadtree policies (the paper's comparison baseline): b = 2
    int b = octree ? 2 : eq1_branching(ln[i].count, s, dims);
    const int kz = dims == 3 ? 1 : 0;
    ln[i].b0 = b;
    ln[i].b = b;
    ln[i].kz = kz;
    for (int l = 0; l < 3; l++)
        ln[i].bx[l] = __ddiv_rn((double)(l == 2 ? bz_of(b, kz) : b), nodes[ln[i].gid].ext[l]);
    ln[i].flag = 1;
    ln[i].halvings = 0;
    ln[i].under = 0;
}

__device__ __forceinline__ int64_t find_node(const LevelNode *ln, int64_t nn, int64_t g) {
    int64_t a = 0, z = nn - 1;  // largest i with cell_base <= g
    while (a < z) {
        int64_t m = (a + z + 1) >> 1;
        if (ln[m].cell_base <= g) a = m; else z = m - 1;
    }
    return a;
}

// ---- A3 + A4: Eq. 2, Eq. 3, histogram ---------------------------------------
// the root level (kRoot) reads the caller's positions directly: every
// particle belongs to node 0 and its record is (pos, caller index)
template <bool kRoot>
__global__ void __launch_bounds__(kThreads) key_hist_kernel(const double4 *__restrict__ act, const int32_t *__restrict__ act_node,
                                                            const double *__restrict__ pos, int64_t n_act,
                                                            const LevelNode *__restrict__ ln,
                                                            const NodeRec *__restrict__ nodes, uint32_t *__restrict__ keys,
                                                            int32_t *__restrict__ hist, int32_t *__restrict__ rank, int round) {
    // (BT_SCATTER_UNROLL particles per thread: independent load chains in flight)
    constexpr int U = BT_SCATTER_UNROLL;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < n_act; p0 += U * stride) {
        int32_t node[U];
        double4 r[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t p = p0 + u * stride;
            if (kRoot) {
                node[u] = p < n_act ? 0 : -1;
                if (node[u] >= 0) r[u] = make_double4(pos[3 * p], pos[3 * p + 1], pos[3 * p + 2], 0.0);
            } else {
                node[u] = p < n_act ? act_node[p] : -1;
                if (node[u] >= 0) r[u] = act[p];
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (node[u] < 0) continue;
            const LevelNode &L = ln[node[u]];
            if (round > 0 && !L.flag) continue;
            const NodeRec &nr = nodes[L.gid];
            const int b = L.b;
            // Eq. 2 (cell_coord_fast: identical results, division only near cell faces)
            const int c1 = cell_coord_fast(r[u].x, nr.lo[0], nr.ext[0], L.bx[0], b);
            const int c2 = cell_coord_fast(r[u].y, nr.lo[1], nr.ext[1], L.bx[1], b);
            const int c3 = cell_coord_fast(r[u].z, nr.lo[2], nr.ext[2], L.bx[2], bz_of(b, L.kz));
            const uint32_t j = (uint32_t)c1 + (uint32_t)c2 * (uint32_t)b + (uint32_t)c3 * (uint32_t)b * (uint32_t)b;
            keys[p0 + u * stride] = (uint32_t)(L.cell_base + j);  // the level's cell index (< 2^32)
#if BT_RANK_HIST
            rank[p0 + u * stride] = atomicAdd(&hist[L.cell_base + j], 1);  // the particle's slot in its cell
#else
            atomicAdd(&hist[L.cell_base + j], 1);
#endif
        }
    }
}

// zero the histogram of nodes that redistribute in this round
__global__ void zero_flagged_kernel(const LevelNode *__restrict__ ln, int64_t nn, int32_t *hist, int64_t ncells) {
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ncells; g += (int64_t)gridDim.x * blockDim.x) {
        int64_t node = find_node(ln, nn, g);
        if (ln[node].flag) hist[g] = 0;
    }
}

// ---- A5: Eq. 4 numerator -----------------------------------------------------
// Warp-uniform loop: every lane runs the same iterations (full-mask ballots).
__global__ void __launch_bounds__(kThreads) under_count_kernel(LevelNode *ln, int64_t nn, const int32_t *__restrict__ hist,
                                                               int64_t ncells, double alpha_s) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < ncells; base += stride) {
        int64_t g = base + threadIdx.x;
        bool under = false;
        int64_t node = 0;
        if (g < ncells) {
            node = find_node(ln, nn, g);
            const LevelNode &L = ln[node];
            int64_t B = (int64_t)L.b * L.b * bz_of(L.b, L.kz);
            under = L.flag && (g - L.cell_base) < B && (double)hist[g] <= alpha_s;
        }
        unsigned m = __ballot_sync(0xffffffffu, under);
        if (under) {  // aggregate per node within the warp (warp-aggregated atomics)
            unsigned same = __match_any_sync(m, (unsigned long long)node);
            int leader = __ffs(same) - 1;
            if ((int)(threadIdx.x & 31) == leader)
                atomicAdd((unsigned long long *)&ln[node].under, (unsigned long long)__popc(same));
        }
    }
}

// r = u / b^3 (Eq. 4); halve iff r >= beta and b > 2 (readings R3, R7)
__global__ void ratio_decide_kernel(LevelNode *ln, int64_t nn, double beta, int *any, const NodeRec *nodes) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nn) return;
    LevelNode &L = ln[i];
    if (!L.flag) return;
    double B = (double)((int64_t)L.b * L.b * bz_of(L.b, L.kz));
    double r = __ddiv_rn((double)L.under, B);
    if (r >= beta && L.b > 2) {
        L.b = max(2, L.b / 2);
        for (int l = 0; l < 3; l++)
            L.bx[l] = __ddiv_rn((double)(l == 2 ? bz_of(L.b, L.kz) : L.b), nodes[L.gid].ext[l]);
        L.halvings++;
        L.under = 0;
        L.flag = 1;
        atomicOr(any, 1);
    } else {
        L.flag = 0;
    }
}

// ---- A6 scan functors ------------------------------------------------------
struct CellIn {
    const int32_t *hist;
    int32_t s;
    bool child_ok;  // depth + 1 < depth_cap
    int octree, dims;
    __device__ CellScan operator()(int64_t g) const {
        long long c = hist[g];
        bool is_node = child_ok && c > s;
        bool is_leaf = c > 0 && !is_node;
        return CellScan{c, is_node ? c : 0, is_node ? node_cells(c, s, octree, dims) : 0, is_node ? 1 : 0,
                        is_leaf ? 1 : 0, is_leaf ? (int)c : 0, 0};
    }
};
struct CellOut {
    int64_t *cpre;
    int32_t *cid;
    int32_t *cact;
    __device__ void operator()(int64_t g, const CellScan &exc, const CellScan &v) const {
        cpre[g] = exc.pre;
        cid[g] = v.nnode ? exc.nnode : (v.nleaf ? exc.nleaf : -1);
        cact[g] = (int32_t)exc.actoff;
    }
};
struct CellsOfNode {
    const LevelNode *ln;
    __device__ long long operator()(int64_t i) const {
        return (long long)ln[i].b0 * ln[i].b0 * bz_of(ln[i].b0, ln[i].kz);
    }
};
struct CellBaseOut {
    LevelNode *ln;
    __device__ void operator()(int64_t i, long long exc, long long) const { ln[i].cell_base = exc; }
};

// ---- A8: children, leaves, cell table --------------------------------------
__global__ void __launch_bounds__(kThreads) emit_kernel(const LevelNode *__restrict__ ln, int64_t nn, int32_t *hist,
                                                        int64_t ncells, const int64_t *__restrict__ cpre,
                                                        const int32_t *__restrict__ cid, const int32_t *__restrict__ cact,
                                                        NodeRec *nodes, int32_t *cells, int64_t cells_base,
                                                        LevelNode *ln_next, int32_t next_gid_base, int32_t *leaf_begin,
                                                        int32_t *leaf_count, int32_t *leaf_depth, int64_t leaf_base,
                                                        int32_t child_depth, int32_t s) {
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ncells; g += (int64_t)gridDim.x * blockDim.x) {
        int64_t node = find_node(ln, nn, g);
        const LevelNode &L = ln[node];
        int32_t c = hist[g];
        int32_t id = cid[g];
        int64_t j = g - L.cell_base;
        int32_t final_pos = L.final_begin + (int32_t)(cpre[g] - cpre[L.cell_base]);
        int32_t code = -1;
        if (id >= 0 && c > 0) {
            // re-derived exactly as in CellIn: ln_next is null at the depth cap
            bool is_node = (c > s) && (ln_next != nullptr);
            if (is_node) {
                int32_t gid = next_gid_base + id;
                LevelNode &C = ln_next[id];
                C.act_begin = cact[g];
                C.count = c;
                C.final_begin = final_pos;
                C.gid = gid;
                const NodeRec &P = nodes[L.gid];
                NodeRec &R = nodes[gid];
                int b = L.b;
                int cc[3] = {(int)(j % b), (int)((j / b) % b), (int)(j / ((int64_t)b * b))};
                for (int l = 0; l < 3; l++) {
                    // child box = equal 1/b slice of the parent (Sec. III-A Step 1); k = 2: whole z slab
                    const double bl = (double)(l == 2 ? bz_of(b, L.kz) : b);
                    double lo = __dadd_rn(P.lo[l], __ddiv_rn(__dmul_rn((double)cc[l], P.ext[l]), bl));
                    double hi = __dadd_rn(P.lo[l], __ddiv_rn(__dmul_rn((double)(cc[l] + 1), P.ext[l]), bl));
                    R.lo[l] = lo;
                    R.ext[l] = __dsub_rn(hi, lo);
                }
                R.depth = child_depth;
                R.b = 0;
                R.cell_base = 0;
                code = node_code(gid);
                // the scatter's cursor: next-level position, bit 31 = child node
                hist[g] = (int32_t)((unsigned)cact[g] | 0x80000000u);
            } else {
                int64_t leaf = leaf_base + id;
                leaf_begin[leaf] = final_pos;
                leaf_count[leaf] = c;
                leaf_depth[leaf] = child_depth;
                code = (int32_t)leaf;
                hist[g] = final_pos;  // the scatter's cursor: final tree position (leaf)
            }
        }
        cells[cells_base + g] = code;
    }
}

// accepted b and global cell base of this level's nodes
__global__ void finalize_level_nodes_kernel(const LevelNode *ln, int64_t nn, NodeRec *nodes, int64_t cells_base,
                                            unsigned long long *halvings) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nn) return;
    NodeRec &R = nodes[ln[i].gid];
    R.b = ln[i].b;
    R.bz = bz_of(R.b, ln[i].kz);
    R.cell_base = cells_base + ln[i].cell_base;
    for (int l = 0; l < 3; l++) R.bx[l] = __ddiv_rn((double)(l == 2 ? R.bz : R.b), R.ext[l]);
    if (ln[i].halvings) atomicAdd(halvings, (unsigned long long)ln[i].halvings);
}

// ---- A7: counting-sort scatter ------------------------------------------------
// Latency-bound per particle (node record -> cell -> returning atomic on the
// cell cursor -> destination): kUnroll particles per thread keep that many
// independent chains in flight.
template <bool kRoot>
__global__ void __launch_bounds__(kThreads) scatter_kernel(const double4 *__restrict__ act, const double *__restrict__ pos,
                                                           int64_t n_act,
                                                           const uint32_t *__restrict__ keys, int32_t *cursor,
                                                           const int32_t *__restrict__ rank,
                                                           double4 *__restrict__ out_final, double4 *__restrict__ act_next) {
    // cursor[g] (written by emit): the cell's next destination, bit 31 set
    // for a child-node cell (next level's active array) -- one returning
    // atomic per particle gives both its slot and its destination array
    constexpr int U = BT_SCATTER_UNROLL;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < n_act; p0 += U * stride) {
        int32_t d[U];
        double4 v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t p = p0 + u * stride;
            if (p < n_act) {
#if BT_RANK_HIST
                d[u] = (int32_t)((unsigned)__ldg(&cursor[keys[p]]) + (unsigned)rank[p]);  // cell start + histogram rank
#else
                d[u] = atomicAdd(&cursor[keys[p]], 1);
#endif
                v[u] = kRoot ? make_double4(pos[3 * p], pos[3 * p + 1], pos[3 * p + 2], __longlong_as_double((long long)p))
                             : act[p];
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (p0 + u * stride >= n_act) continue;
            const int32_t dst = (int32_t)((unsigned)d[u] & 0x7fffffffu);
            if (d[u] < 0) act_next[dst] = v[u];  // (its node id: node_ids_kernel, coalesced)
            else out_final[dst] = v[u];
        }
    }
}

// next level's node id of every active position: one warp per node writes its
// contiguous range (instead of a random 4-byte store per particle in the scatter)
__global__ void node_ids_kernel(const LevelNode *__restrict__ ln, int64_t nn, int32_t *__restrict__ act_node) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nn; i += warps) {
        const int32_t b = ln[i].act_begin, c = ln[i].count;
        for (int32_t k = lane; k < c; k += 32) act_node[b + k] = (int32_t)i;
    }
}

// ---- A9: per-leaf canonical order (ascending caller index) + tight box -------
// Exact fp64 warp min / max through order-preserving 64-bit keys (sign bit
// flipped for positives, all bits for negatives; no NaN here): two 32-bit
// redux.sync per value instead of five shuffle + DMNMX steps.
__device__ __forceinline__ unsigned long long dkey(double d) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(d);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dunkey(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}
__device__ __forceinline__ unsigned long long warp_min_key(unsigned long long k) {
    const unsigned hi = __reduce_min_sync(0xffffffffu, (unsigned)(k >> 32));
    const unsigned lo = __reduce_min_sync(0xffffffffu, ((unsigned)(k >> 32) == hi) ? (unsigned)k : 0xffffffffu);
    return ((unsigned long long)hi << 32) | lo;
}
__device__ __forceinline__ unsigned long long warp_max_key(unsigned long long k) {
    const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(k >> 32));
    const unsigned lo = __reduce_max_sync(0xffffffffu, ((unsigned)(k >> 32) == hi) ? (unsigned)k : 0u);
    return ((unsigned long long)hi << 32) | lo;
}

// One warp per leaf.  rank(e) = #{k in leaf : idx_k < idx_e} (caller indices
// are distinct), O(m^2 / 32) per leaf: m <= s = 64 in the configurations.
// Leaves above kBigLeaf particles (only at the depth cap, R14: e.g. many
// coincident points) get their box here and their order from a segmented
// radix sort afterwards (big_leaf_*), which keeps the build O(m log m).
constexpr int kBigLeaf = 1024;
__global__ void __launch_bounds__(kThreads) leaf_finalize_kernel(const double4 *__restrict__ src, double4 *__restrict__ dst,
                                                                 float4 *__restrict__ dst32, int32_t *__restrict__ perm,
                                                                 const int32_t *__restrict__ leaf_begin,
                                                                 const int32_t *__restrict__ leaf_count, int64_t n_leaves,
                                                                 double *__restrict__ leaf_box,
                                                                 unsigned long long *max_leaf, int32_t s) {
    int lane = threadIdx.x & 31;
    int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int wmax = 0, wover = 0;
    for (int64_t L = warp; L < n_leaves; L += nwarps) {
        int32_t b0 = leaf_begin[L], m = leaf_count[L];
        if (m <= 64) {
            // single pass, the leaf's records in registers (one or two per lane)
            const bool two = m > 32;
            const bool ok0 = lane < m, ok1 = two && lane + 32 < m;
            const double4 v0 = ok0 ? src[b0 + lane] : make_double4(0, 0, 0, 0);
            const double4 v1 = ok1 ? src[b0 + 32 + lane] : make_double4(0, 0, 0, 0);
            // tight box: exact min / max (keys of absent slots: +inf / -inf)
            const unsigned long long KMAX = dkey(INFINITY), KMIN = dkey(-INFINITY);
            double c[3];
            for (int l = 0; l < 3; l++) {
                const double x0 = l == 0 ? v0.x : (l == 1 ? v0.y : v0.z);
                const double x1 = l == 0 ? v1.x : (l == 1 ? v1.y : v1.z);
                const unsigned long long k0 = dkey(x0), k1 = dkey(x1);
                unsigned long long kmin = ok0 ? k0 : KMAX, kmax = ok0 ? k0 : KMIN;
                if (ok1) {
                    kmin = min(kmin, k1);
                    kmax = max(kmax, k1);
                }
                const double a = dunkey(warp_min_key(kmin)), b = dunkey(warp_max_key(kmax));
                if (lane == 0) { leaf_box[6 * L + l] = a; leaf_box[6 * L + 3 + l] = b; }
                c[l] = 0.5 * (a + b);  // leaf centre for the compact fp32 records
            }
            // canonical order: rank(e) = #{k : idx_k < idx_e} (caller indices < 2^31, distinct)
            const int i0 = ok0 ? (int)__double_as_longlong(v0.w) : 0x7fffffff;
            const int i1 = ok1 ? (int)__double_as_longlong(v1.w) : 0x7fffffff;
            int r0 = 0, r1 = 0;
            if (!two) {
                for (int j = 0; j < m; j++) r0 += __shfl_sync(0xffffffffu, i0, j) < i0;
            } else {
                for (int j = 0; j < 32; j++) {
                    const int o0 = __shfl_sync(0xffffffffu, i0, j), o1 = __shfl_sync(0xffffffffu, i1, j);
                    r0 += (o0 < i0) + (o1 < i0);
                    r1 += (o0 < i1) + (o1 < i1);
                }
            }
            if (ok0) {
                dst[b0 + r0] = v0;
                perm[b0 + r0] = i0;
                dst32[b0 + r0] = make_float4(__double2float_rn(__dsub_rn(v0.x, c[0])), __double2float_rn(__dsub_rn(v0.y, c[1])),
                                             __double2float_rn(__dsub_rn(v0.z, c[2])), __int_as_float(i0));
            }
            if (ok1) {
                dst[b0 + r1] = v1;
                perm[b0 + r1] = i1;
                dst32[b0 + r1] = make_float4(__double2float_rn(__dsub_rn(v1.x, c[0])), __double2float_rn(__dsub_rn(v1.y, c[1])),
                                             __double2float_rn(__dsub_rn(v1.z, c[2])), __int_as_float(i1));
            }
            wmax = max(wmax, m);
            wover += (m > s) ? 1 : 0;  // over-full leaf (depth cap, R14)
            continue;
        }
        // tight box (exact fp64 min / max)
        double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int32_t e = lane; e < m; e += 32) {
            const double4 v = src[b0 + e];
            mn[0] = fmin(mn[0], v.x); mn[1] = fmin(mn[1], v.y); mn[2] = fmin(mn[2], v.z);
            mx[0] = fmax(mx[0], v.x); mx[1] = fmax(mx[1], v.y); mx[2] = fmax(mx[2], v.z);
        }
        double c[3];
        for (int l = 0; l < 3; l++) {
            double a = mn[l], b = mx[l];
            for (int d = 16; d; d >>= 1) {
                a = fmin(a, __shfl_xor_sync(0xffffffffu, a, d));
                b = fmax(b, __shfl_xor_sync(0xffffffffu, b, d));
            }
            if (lane == 0) { leaf_box[6 * L + l] = a; leaf_box[6 * L + 3 + l] = b; }
            c[l] = 0.5 * (a + b);  // leaf centre for the compact fp32 records
        }
        wmax = max(wmax, m);
        wover += (m > s) ? 1 : 0;
        if (m > kBigLeaf) continue;  // ordered by big_leaf_write_kernel
        // canonical order: rank(e) = #{k : idx_k < idx_e}
        for (int32_t e0 = 0; e0 < m; e0 += 32) {
            int32_t e = e0 + lane;
            double4 v = make_double4(0, 0, 0, 0);
            long long my = 0x7fffffffffffffffLL;
            if (e < m) {
                v = src[b0 + e];
                my = __double_as_longlong(v.w);
            }
            int32_t rank = 0;
            for (int32_t k0 = 0; k0 < m; k0 += 32) {
                long long o = 0x7fffffffffffffffLL;
                if (k0 + lane < m) o = __double_as_longlong(src[b0 + k0 + lane].w);
                int lim = min(32, m - k0);
                for (int q = 0; q < lim; q++) {
                    long long ok = __shfl_sync(0xffffffffu, o, q);
                    rank += (ok < my);
                }
            }
            if (e < m) {
                dst[b0 + rank] = v;
                // compact record: fl32(fl64(x - c_L)), caller index (walk staging, lemma L4)
                perm[b0 + rank] = (int32_t)my;
                dst32[b0 + rank] = make_float4(__double2float_rn(__dsub_rn(v.x, c[0])),
                                               __double2float_rn(__dsub_rn(v.y, c[1])),
                                               __double2float_rn(__dsub_rn(v.z, c[2])), __int_as_float((int)my));
            }
        }
    }
    // one atomic per warp (a per-leaf atomic on one address serialises 10^6 updates)
    if (lane == 0 && wmax > 0) {
        atomicMax(max_leaf, (unsigned long long)wmax);
        if (wover) atomicAdd(max_leaf + 1, (unsigned long long)wover);
    }
}

// ---- leaves renumbered in depth-first order (ascending tree position) -------
__global__ void mark_leaf_begin_kernel(const int32_t *begin, int64_t n_leaves, int32_t *flag) {
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < n_leaves; L += (int64_t)gridDim.x * blockDim.x)
        flag[begin[L]] = 1;
}
struct FlagIn {
    const int32_t *f;
    __device__ int operator()(int64_t i) const { return f[i]; }
};
struct FlagOut {
    int32_t *excl;
    __device__ void operator()(int64_t i, int exc, int) const { excl[i] = exc; }
};
__global__ void permute_leaves_kernel(const int32_t *excl, int64_t n_leaves, const int32_t *b0, const int32_t *c0,
                                      const int32_t *d0, int32_t *b1, int32_t *c1, int32_t *d1, int32_t *map) {
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < n_leaves; L += (int64_t)gridDim.x * blockDim.x) {
        int32_t nid = excl[b0[L]];
        b1[nid] = b0[L];
        c1[nid] = c0[L];
        d1[nid] = d0[L];
        map[L] = nid;
    }
}
__global__ void remap_cells_kernel(int32_t *cells, int64_t n_cells, const int32_t *map) {
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_cells; g += (int64_t)gridDim.x * blockDim.x) {
        int32_t c = cells[g];
        if (c >= 0) cells[g] = map[c];
    }
}

// ---- walk unit order: Morton (Z-order) of the leaf centre ------------------
// The walk processes units in array order; depth-first leaf order puts the
// +z neighbour of a root cell b^2 cells later, so concurrently processed units
// would not share candidate leaves in L2.  Units are bucketed by the top
// bits (about 2 buckets per unit, at most 21) of the 30-bit Morton code of
// their leaf centre (counting sort).
constexpr int kMortonBits = 21;  // at most; fewer for few units (about 2 buckets per unit)

__device__ __forceinline__ unsigned spread3(unsigned v) {  // 10 bits -> every third bit
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000ffu;
    v = (v | (v << 8)) & 0x0300f00fu;
    v = (v | (v << 4)) & 0x030c30c3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

// per-leaf staging record: centre (the same 0.5 (lo + hi) as the compact
// records), half-extent, begin, count
// ---- leaves above kBigLeaf particles: segmented sort by caller index -------
__global__ void big_leaf_list_kernel(const int32_t *__restrict__ begin, const int32_t *__restrict__ count, int64_t n_leaves,
                                     int32_t *__restrict__ ids, int32_t *__restrict__ seg_b, int32_t *__restrict__ seg_e,
                                     int *n_big) {
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < n_leaves; L += (int64_t)gridDim.x * blockDim.x)
        if (count[L] > kBigLeaf) {
            const int k = atomicAdd(n_big, 1);
            ids[k] = (int32_t)L;
            seg_b[k] = begin[L];
            seg_e[k] = begin[L] + count[L];
        }
}
// keys = caller index, values = position, over each big leaf's positions (one block per leaf)
__global__ void big_leaf_keys_kernel(const double4 *__restrict__ src, const int32_t *__restrict__ seg_b,
                                     const int32_t *__restrict__ seg_e, int nbig, int32_t *__restrict__ key,
                                     int32_t *__restrict__ val) {
    for (int k = blockIdx.x; k < nbig; k += gridDim.x)
        for (int32_t p = seg_b[k] + threadIdx.x; p < seg_e[k]; p += blockDim.x) {
            key[p] = (int32_t)__double_as_longlong(src[p].w);
            val[p] = p;
        }
}
// records of each big leaf in ascending caller index (compact records relative to its centre)
__global__ void big_leaf_write_kernel(const double4 *__restrict__ src, const int32_t *__restrict__ ids,
                                      const int32_t *__restrict__ seg_b, const int32_t *__restrict__ seg_e, int nbig,
                                      const int32_t *__restrict__ val, const double *__restrict__ leaf_box,
                                      double4 *__restrict__ dst, float4 *__restrict__ dst32, int32_t *__restrict__ perm) {
    for (int k = blockIdx.x; k < nbig; k += gridDim.x) {
        const double *bx = leaf_box + 6 * (int64_t)ids[k];
        const double c0 = 0.5 * (bx[0] + bx[3]), c1 = 0.5 * (bx[1] + bx[4]), c2 = 0.5 * (bx[2] + bx[5]);
        for (int32_t p = seg_b[k] + threadIdx.x; p < seg_e[k]; p += blockDim.x) {
            const double4 v = src[val[p]];
            const int i = (int)__double_as_longlong(v.w);
            dst[p] = v;
            perm[p] = i;
            dst32[p] = make_float4(__double2float_rn(__dsub_rn(v.x, c0)), __double2float_rn(__dsub_rn(v.y, c1)),
                                   __double2float_rn(__dsub_rn(v.z, c2)), __int_as_float(i));
        }
    }
}

__global__ void leaf_rec_kernel(const double *__restrict__ box, const int32_t *__restrict__ begin,
                                const int32_t *__restrict__ count, int64_t nl, LeafRec *__restrict__ out) {
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < nl; L += (int64_t)gridDim.x * blockDim.x) {
        const double *b = box + 6 * L;
        LeafRec r;
        r.cx = 0.5 * (b[0] + b[3]);
        r.cy = 0.5 * (b[1] + b[4]);
        r.cz = 0.5 * (b[2] + b[5]);
        r.H = 0.5 * fmax(fmax(b[3] - b[0], b[4] - b[1]), b[5] - b[2]);
        r.begin = begin[L];
        r.count = count[L];
        r.pad_[0] = r.pad_[1] = 0;
        out[L] = r;
    }
}

__global__ void unit_key_kernel(const int4 *__restrict__ units, const long long *__restrict__ dnu,
                                const double *__restrict__ leaf_box, const double *__restrict__ box, int mbits,
                                unsigned *__restrict__ key, int32_t *__restrict__ hist) {
    const int64_t nu = *dnu;  // (the unit count stays on the device: grids sized by its bound)
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nu; u += (int64_t)gridDim.x * blockDim.x) {
        const double *lb = leaf_box + 6 * (int64_t)units[u].x;
        unsigned q[3];
        for (int l = 0; l < 3; l++) {
            const double c = 0.5 * (lb[l] + lb[3 + l]);
            const double f = (c - box[l]) / (box[3 + l] - box[l]);
            q[l] = (unsigned)fmin(1023.0, fmax(0.0, f * 1024.0));
        }
        const unsigned m = spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2);
        const unsigned k = m >> (30 - mbits);
        key[u] = k;
        atomicAdd(&hist[k], 1);
    }
}

struct HistIn {
    const int32_t *h;
    __device__ long long operator()(int64_t i) const { return h[i]; }
};
struct HistOut {
    int32_t *start;
    __device__ void operator()(int64_t i, long long exc, long long) const { start[i] = (int32_t)exc; }
};

__global__ void unit_scatter_kernel(const int4 *__restrict__ units, const long long *__restrict__ dnu,
                                    const unsigned *__restrict__ key, int32_t *__restrict__ cursor,
                                    int4 *__restrict__ out) {
    const int64_t nu = *dnu;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nu; u += (int64_t)gridDim.x * blockDim.x)
        out[atomicAdd(&cursor[key[u]], 1)] = units[u];
}

constexpr int kUnitQ = 64;  // queries per walk work unit
#ifndef BT_SMALL_LEAF
#define BT_SMALL_LEAF 16
#endif
constexpr int kSmallLeaf = BT_SMALL_LEAF;  // leaves this small are paired into one unit

// Work units (the paper's "blocked approach", Sec. IV-E; reading R16):
// one unit per leaf (leaves above 64 split into 64-query units), except that
// consecutive small leaves (<= 16 particles, adjacent in depth-first order,
// whose union box is at most twice as wide as the wider of the two) are
// paired: a descent and a staging pass per leaf would otherwise serve only a
// handful of queries.  Runs of small leaves pair (0,1), (2,3), ... by rank.
struct MaxScan {
    long long v;
    __host__ __device__ MaxScan operator+(const MaxScan &o) const { return MaxScan{v > o.v ? v : o.v}; }
};
struct RunStartIn {
    const int32_t *cnt;
    __device__ MaxScan operator()(int64_t L) const {
        const bool cont = L > 0 && cnt[L] <= kSmallLeaf && cnt[L - 1] <= kSmallLeaf;
        return MaxScan{cont ? 0 : L};
    }
};
struct RunStartOut {
    int32_t *rs;
    __device__ void operator()(int64_t L, const MaxScan &exc, const MaxScan &v) const {
        rs[L] = (int32_t)(exc.v > v.v ? exc.v : v.v);  // inclusive max
    }
};

__global__ void pair_leaves_kernel(const int32_t *__restrict__ cnt, const double *__restrict__ box,
                                   const int32_t *__restrict__ rs, int64_t nl, int32_t *__restrict__ merge) {
    for (int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; L < nl; L += (int64_t)gridDim.x * blockDim.x) {
        int m = 0;
        if (L + 1 < nl && cnt[L] <= kSmallLeaf && cnt[L + 1] <= kSmallLeaf && rs[L + 1] == rs[L] &&
            ((L - rs[L]) & 1) == 0) {
            const double *a = box + 6 * L, *b = box + 6 * (L + 1);
            double wa = 0.0, wb = 0.0, wu = 0.0;
            for (int l = 0; l < 3; l++) {
                wa = fmax(wa, a[3 + l] - a[l]);
                wb = fmax(wb, b[3 + l] - b[l]);
                wu = fmax(wu, fmax(a[3 + l], b[3 + l]) - fmin(a[l], b[l]));
            }
            m = wu <= 2.0 * fmax(wa, wb) ? 1 : 0;
        }
        merge[L] = m;
    }
}

struct UnitsOfLeaf {
    const int32_t *cnt;
    const int32_t *merge;
    __device__ long long operator()(int64_t L) const {
        if (L > 0 && merge[L - 1]) return 0;  // paired into the previous leaf's unit
        const int q = cnt[L] + (merge[L] ? cnt[L + 1] : 0);
        return (q + kUnitQ - 1) / kUnitQ;
    }
};
struct NullOut {
    __device__ void operator()(int64_t, long long, long long) const {}
};
struct UnitsOut {
    const int32_t *begin;
    const int32_t *cnt;
    const int32_t *merge;
    int4 *units;
    __device__ void operator()(int64_t L, long long exc, long long v) const {
        const int q = cnt[L] + ((v > 0 && merge[L]) ? cnt[L + 1] : 0);
        for (long long u = 0; u < v; u++) {
            int q0 = (int)(u * kUnitQ);
            units[exc + u] = make_int4((int)L, begin[L] + q0, min(kUnitQ, q - q0), 0);
        }
    }
};

}  // namespace

// Leaves above kBigLeaf particles (depth cap): canonical order by a segmented
// radix sort of their caller indices (cub), then their records are written.
void order_big_leaves(TreeDev &t, const double4 *fin, int *dcount) {
    cudaStream_t st = stream();
    const int64_t n = t.n;
    DBuf<int32_t> ids(t.n_leaves), sb(t.n_leaves), se(t.n_leaves);
    BT_CUDA(cudaMemsetAsync(dcount, 0, sizeof(int), st));
    big_leaf_list_kernel<<<grid_for(t.n_leaves, kThreads, (int64_t)num_sms() * 8), kThreads, 0, st>>>(
        t.leaf_begin.p, t.leaf_count.p, t.n_leaves, ids.p, sb.p, se.p, dcount);
    BT_LAUNCH("big_leaf_list");
    int nbig = 0;
    read_back({{dcount, &nbig, sizeof(int)}});
    if (nbig == 0) return;
    DBuf<int32_t> kin(n), kout(n), vin(n), vout(n);
    const unsigned gb = (unsigned)std::min<int64_t>(nbig, (int64_t)num_sms() * 8);
    big_leaf_keys_kernel<<<gb, kThreads, 0, st>>>(fin, sb.p, se.p, nbig, kin.p, vin.p);
    BT_LAUNCH("big_leaf_keys");
    size_t tmp_bytes = 0;
    BT_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, tmp_bytes, kin.p, kout.p, vin.p, vout.p, (int)n, nbig, sb.p,
                                                se.p, st));
    DBuf<unsigned char> tmp(tmp_bytes > 0 ? tmp_bytes : 1);
    BT_CUDA(cub::DeviceSegmentedSort::SortPairs(tmp.p, tmp_bytes, kin.p, kout.p, vin.p, vout.p, (int)n, nbig, sb.p,
                                                se.p, st));
    big_leaf_write_kernel<<<gb, kThreads, 0, st>>>(fin, ids.p, sb.p, se.p, nbig, vout.p, t.leaf_box.p, t.rec.p,
                                                   t.rec32.p, t.perm.p);
    BT_LAUNCH("big_leaf_write");
}

// ---------------------------------------------------------------------------
// Host driver (K12): level loop.  Reads back a few scalars per level (total
// cells, any-halving flag per round, next-level totals).
// ---------------------------------------------------------------------------
void build_tree(TreeDev &t, const double *pos) {
    const int64_t n = t.n;
    cudaStream_t st = stream();
    t.n_nodes = t.n_cells = t.n_leaves = t.n_units = 0;
    t.depth = 0;
    t.root_b = 0;
    t.halvings = t.overfull = t.max_leaf = 0;
    t.root_is_leaf = true;
    if (n == 0) {
        t.M = 0;
        for (int l = 0; l < 3; l++) t.box_lo[l] = t.box_hi[l] = 0;
        return;
    }
    const int sms = num_sms();
    const unsigned gridN = grid_for(n, kThreads, (int64_t)sms * 16);

    DBuf<double4> act[2];
    DBuf<int32_t> act_node[2];
    DBuf<double4> fin;
    DBuf<int> dflags;
    DBuf<unsigned long long> dstat;  // halvings, max_leaf, overfull
    DBuf<double> partials, dbox;
    DBuf<long long> dnu(1);  // work units (A9), read with the build's closing read
    int64_t max_leaf_h = n;  // largest leaf (the root leaf: n; else from the levels' cell scans)
    {
        Phase ph("build.setup");
        fin.alloc(n);
        t.rec.alloc(n);
        dflags.alloc(4);
        dstat.alloc(4);
        BT_CUDA(cudaMemsetAsync(dflags.p, 0, 4 * sizeof(int), st));
        BT_CUDA(cudaMemsetAsync(dstat.p, 0, 4 * sizeof(unsigned long long), st));
        partials.alloc(6 * (size_t)gridN);
        dbox.alloc(8);
        t.nodes.reserve(1024, 0);
    }

    // A1: records in caller order + root box
    {
        Phase ph("build.bbox");
        // records are written only for a root leaf (straight into the final
        // array); otherwise the root level reads pos itself
        const bool root_leaf = n <= t.s || t.depth_cap == 0;
        pack_bbox_kernel<<<gridN, kThreads, 0, st>>>(pos, n, root_leaf ? fin.p : nullptr, partials.p, dflags.p);
        BT_LAUNCH("pack_bbox");
        root_box_kernel<<<1, 256, 0, st>>>(partials.p, (int)gridN, t.nodes.p, dbox.p);
        BT_LAUNCH("root_box");
        // (box, M and the input check are read back with the build's last
        // control read: no host round trip here)
    }

    // Root is a leaf when n <= s or the depth cap is 0.
    if (n <= t.s || t.depth_cap == 0) {
        t.leaf_begin.alloc(1);
        t.leaf_count.alloc(1);
        t.leaf_depth.alloc(1);
        int32_t hl[3] = {0, (int32_t)n, 0};
        BT_CUDA(cudaMemcpyAsync(t.leaf_begin.p, &hl[0], 4, cudaMemcpyHostToDevice, st));
        BT_CUDA(cudaMemcpyAsync(t.leaf_count.p, &hl[1], 4, cudaMemcpyHostToDevice, st));
        BT_CUDA(cudaMemcpyAsync(t.leaf_depth.p, &hl[2], 4, cudaMemcpyHostToDevice, st));
        t.n_leaves = 1;
        t.n_nodes = 0;
        t.level_begin.clear();
        t.level_cells.clear();
        t.root_is_leaf = true;
    } else {
        t.root_is_leaf = false;
        max_leaf_h = 0;
        act[0].alloc(n);
        act_node[0].alloc(n);  // (level 0 reads pos and node 0: neither array)
        act[1].alloc(n);
        act_node[1].alloc(n);
        DBuf<uint32_t> keys(n);
        DBuf<int32_t> ranks(BT_RANK_HIST ? n : 1);
        DBuf<LevelNode> ln(1), ln_next;
        {
            LevelNode r{};
            r.act_begin = 0;
            r.count = (int32_t)n;
            r.final_begin = 0;
            r.gid = 0;
            BT_CUDA(cudaMemcpyAsync(ln.p, &r, sizeof(r), cudaMemcpyHostToDevice, st));
        }
        t.n_nodes = 1;
        t.level_begin.assign(1, 0);
        t.level_cells.assign(1, 0);
        t.leaf_begin.reserve(1024, 0);
        t.leaf_count.reserve(1024, 0);
        t.leaf_depth.reserve(1024, 0);
        int64_t nn = 1, n_act = n;
        int cur = 0;
        int level = 0;
        DBuf<int32_t> hist;
        DBuf<int64_t> cpre;
        DBuf<int32_t> cid, cact;
        DBuf<CellScan> dcs(1);
        // the level's cell count: the root's from Eq. 1 on the host, every
        // later level's from the previous level's cell scan (ncnext) -- one
        // host read per level (its cell scan + the halving flag of round 0)
        int64_t ncells_next = node_cells(n, t.s, t.octree ? 1 : 0, t.dims);
        while (nn > 0) {
            Phase ph("build.level");
            // A2: Eq. 1 and the level's cell layout
            level_b_kernel<<<grid_for(nn, kThreads), kThreads, 0, st>>>(ln.p, nn, t.s, t.octree ? 1 : 0, t.dims,
                                                                        t.nodes.p);
            BT_LAUNCH("level_b");
            device_scan<long long>(CellsOfNode{ln.p}, CellBaseOut{ln.p}, nn, (long long *)nullptr);
            const int64_t ncells = ncells_next;
            if (ncells > (int64_t)0xffffffffLL)  // (keys hold a level's cell index in 32 bits)
                throw Error(BT_ERR_OOM, "bt_build: more than 2^32 sub-cells in one level (bucket_size too small for n)");
            hist.reserve(ncells, 0);
            cpre.reserve(ncells, 0);
            cid.reserve(ncells, 0);
            cact.reserve(ncells, 0);
            t.cells.reserve(t.n_cells + ncells, t.n_cells);
            BT_CUDA(cudaMemsetAsync(hist.p, 0, ncells * sizeof(int32_t), st));
            const unsigned gridC = grid_for(ncells, kThreads, (int64_t)sms * 16);
            const unsigned gridA = grid_for(n_act, kThreads, (int64_t)sms * 16);

            // A3-A5: distribute, ratio, halving rounds (at most log2 b0 rounds).
            // Round 0 is followed by the level's cell scan (A6) before the
            // host looks at its halving flag: when no node halves (the common
            // case) that scan is the level's and one read returns both.
            const bool child_ok = (level + 1) < t.depth_cap;
            const CellIn cin{hist.p, (int32_t)t.s, child_ok, t.octree ? 1 : 0, t.dims};
            CellScan tot{};
            bool scanned = false;
            for (int round = 0;; round++) {
                if (round > 0) {
                    zero_flagged_kernel<<<gridC, kThreads, 0, st>>>(ln.p, nn, hist.p, ncells);
                    BT_LAUNCH("zero_flagged");
                }
                if (level == 0)
                    key_hist_kernel<true><<<gridA, kThreads, 0, st>>>(nullptr, nullptr, pos, n_act, ln.p, t.nodes.p,
                                                                      keys.p, hist.p, ranks.p, round);
                else
                    key_hist_kernel<false><<<gridA, kThreads, 0, st>>>(act[cur].p, act_node[cur].p, nullptr, n_act, ln.p,
                                                                       t.nodes.p, keys.p, hist.p, ranks.p, round);
                BT_LAUNCH("key_hist");
                if (t.octree) break;  // no ratio test for the octree policy
                under_count_kernel<<<gridC, kThreads, 0, st>>>(ln.p, nn, hist.p, ncells, t.alpha * (double)t.s);
                BT_LAUNCH("under_count");
                BT_CUDA(cudaMemsetAsync(dflags.p + 1, 0, sizeof(int), st));
                ratio_decide_kernel<<<grid_for(nn, kThreads), kThreads, 0, st>>>(ln.p, nn, t.beta, dflags.p + 1, t.nodes.p);
                BT_LAUNCH("ratio_decide");
                int any = 0;
                if (round == 0) {
                    device_scan<CellScan>(cin, CellOut{cpre.p, cid.p, cact.p}, ncells, dcs.p);
                    read_back({{dflags.p + 1, &any, sizeof(int)}, {dcs.p, &tot, sizeof(CellScan)}});
                    scanned = !any;
                } else {
                    read_back({{dflags.p + 1, &any, sizeof(int)}});
                }
                if (!any) break;
            }
            finalize_level_nodes_kernel<<<grid_for(nn, kThreads), kThreads, 0, st>>>(ln.p, nn, t.nodes.p, t.n_cells,
                                                                                       dstat.p);
            BT_LAUNCH("finalize_level_nodes");

            // A6: one scan over the level's cells (done above unless a node halved)
            if (!scanned) {
                device_scan<CellScan>(cin, CellOut{cpre.p, cid.p, cact.p}, ncells, dcs.p);
                read_back({{dcs.p, &tot, sizeof(CellScan)}});
            }
            const int64_t nn_next = tot.nnode, n_act_next = tot.actoff, nleaf = tot.nleaf;
            ncells_next = tot.ncnext;
            max_leaf_h = std::max<int64_t>(max_leaf_h, tot.maxleaf);

            // A8: emit children / leaves / cell table
            ln_next.alloc(nn_next > 0 ? nn_next : 1);
            t.nodes.reserve(t.n_nodes + nn_next, t.n_nodes);
            t.leaf_begin.reserve(t.n_leaves + nleaf, t.n_leaves);
            t.leaf_count.reserve(t.n_leaves + nleaf, t.n_leaves);
            t.leaf_depth.reserve(t.n_leaves + nleaf, t.n_leaves);
            emit_kernel<<<gridC, kThreads, 0, st>>>(ln.p, nn, hist.p, ncells, cpre.p, cid.p, cact.p, t.nodes.p, t.cells.p,
                                                    t.n_cells, child_ok ? ln_next.p : nullptr, (int32_t)t.n_nodes,
                                                    t.leaf_begin.p, t.leaf_count.p, t.leaf_depth.p, t.n_leaves,
                                                    level + 1, t.s);
            BT_LAUNCH("emit");

            // A7: scatter (cursors initialised by emit in the histogram).  (A two-pass variant --
            // particles first grouped by coarse cell range so the scatter's
            // destination window stays L2-resident -- measured slower in round 2:
            // cfg 5 levels 3.9 -> 5.1 ms.)
            if (level == 0)
                scatter_kernel<true><<<gridA, kThreads, 0, st>>>(nullptr, pos, n_act, keys.p, hist.p, ranks.p, fin.p,
                                                                 act[cur ^ 1].p);
            else
                scatter_kernel<false><<<gridA, kThreads, 0, st>>>(act[cur].p, nullptr, n_act, keys.p, hist.p, ranks.p, fin.p,
                                                                  act[cur ^ 1].p);
            BT_LAUNCH("scatter");
            if (nn_next > 0) {
                node_ids_kernel<<<grid_for(nn_next * 32, kThreads, (int64_t)sms * 16), kThreads, 0, st>>>(
                    ln_next.p, nn_next, act_node[cur ^ 1].p);
                BT_LAUNCH("node_ids");
            }

            if (nleaf > 0) t.depth = level + 1;
            t.n_cells += ncells;
            t.level_cells.push_back(t.n_cells);
            t.n_leaves += nleaf;
            if (nn_next > 0) t.level_begin.push_back(t.n_nodes);  // the next depth's node ids start here
            t.n_nodes += nn_next;
            std::swap(ln, ln_next);
            nn = nn_next;
            n_act = n_act_next;
            cur ^= 1;
            level++;
        }
        t.level_begin.push_back(t.n_nodes);
    }

    // Leaves were numbered level by level; renumber them in depth-first order
    // (ascending first tree position), which is the paper's walk order.
    if (!t.root_is_leaf) {
        Phase ph("build.leaf_order");
        DBuf<int32_t> flag(n), excl(n), map(t.n_leaves);
        DBuf<int32_t> b1(t.n_leaves), c1(t.n_leaves), d1(t.n_leaves);
        BT_CUDA(cudaMemsetAsync(flag.p, 0, n * sizeof(int32_t), st));
        mark_leaf_begin_kernel<<<grid_for(t.n_leaves, kThreads, (int64_t)sms * 16), kThreads, 0, st>>>(
            t.leaf_begin.p, t.n_leaves, flag.p);
        BT_LAUNCH("mark_leaf_begin");
        device_scan<int>(FlagIn{flag.p}, FlagOut{excl.p}, n, (int *)nullptr);
        permute_leaves_kernel<<<grid_for(t.n_leaves, kThreads, (int64_t)sms * 16), kThreads, 0, st>>>(
            excl.p, t.n_leaves, t.leaf_begin.p, t.leaf_count.p, t.leaf_depth.p, b1.p, c1.p, d1.p, map.p);
        BT_LAUNCH("permute_leaves");
        remap_cells_kernel<<<grid_for(t.n_cells, kThreads, (int64_t)sms * 16), kThreads, 0, st>>>(t.cells.p, t.n_cells,
                                                                                                  map.p);
        BT_LAUNCH("remap_cells");
        t.leaf_begin = std::move(b1);
        t.leaf_count = std::move(c1);
        t.leaf_depth = std::move(d1);
    }

    // A9: canonical leaf order + tight boxes; work units
    {
        Phase ph("build.leaves");
        t.leaf_box.alloc(6 * (size_t)t.n_leaves);
        t.rec32.alloc(n);
        t.perm.alloc(n);
        leaf_finalize_kernel<<<grid_for(t.n_leaves * 32, kThreads, (int64_t)sms * 32), kThreads, 0, st>>>(
            fin.p, t.rec.p, t.rec32.p, t.perm.p, t.leaf_begin.p, t.leaf_count.p, t.n_leaves, t.leaf_box.p, dstat.p + 1, t.s);
        BT_LAUNCH("leaf_finalize");
        t.leaf_rec.alloc(t.n_leaves);
        leaf_rec_kernel<<<grid_for(t.n_leaves, kThreads, (int64_t)sms * 8), kThreads, 0, st>>>(
            t.leaf_box.p, t.leaf_begin.p, t.leaf_count.p, t.n_leaves, t.leaf_rec.p);
        BT_LAUNCH("leaf_rec");
        // small leaves paired (runs of small leaves, pair by rank, box check)
        DBuf<int32_t> rs(t.n_leaves), merge(t.n_leaves);
        device_scan<MaxScan>(RunStartIn{t.leaf_count.p}, RunStartOut{rs.p}, t.n_leaves, (MaxScan *)nullptr);
        pair_leaves_kernel<<<grid_for(t.n_leaves, kThreads, (int64_t)sms * 8), kThreads, 0, st>>>(
            t.leaf_count.p, t.leaf_box.p, rs.p, t.n_leaves, merge.p);
        BT_LAUNCH("pair_leaves");
        // leaves above kBigLeaf (depth cap): records in canonical order by a segmented sort
        if (max_leaf_h > kBigLeaf) order_big_leaves(t, fin.p, dflags.p + 2);
        // units, sized by their bound (<= ceil(q / kUnitQ) per leaf): the count
        // stays on the device until the build's closing read
        const int64_t nu_bound = t.n_leaves + n / kUnitQ + 1;
        DBuf<int4> units_raw(nu_bound);
        t.units.alloc(nu_bound);
        device_scan<long long>(UnitsOfLeaf{t.leaf_count.p, merge.p},
                               UnitsOut{t.leaf_begin.p, t.leaf_count.p, merge.p, units_raw.p}, t.n_leaves, dnu.p);
        {  // Morton order of the units (walk locality)
            DBuf<unsigned> key(nu_bound);
            int mbits = 6;
            while (mbits < kMortonBits && (int64_t(1) << mbits) < 2 * nu_bound) mbits++;
            DBuf<int32_t> bucket(size_t(1) << mbits);
            BT_CUDA(cudaMemsetAsync(bucket.p, 0, sizeof(int32_t) << mbits, st));
            unit_key_kernel<<<grid_for(nu_bound, kThreads, (int64_t)sms * 8), kThreads, 0, st>>>(
                units_raw.p, dnu.p, t.leaf_box.p, dbox.p, mbits, key.p, bucket.p);
            BT_LAUNCH("unit_key");
            device_scan<long long>(HistIn{bucket.p}, HistOut{bucket.p}, int64_t(1) << mbits, (long long *)nullptr);
            unit_scatter_kernel<<<grid_for(nu_bound, kThreads, (int64_t)sms * 8), kThreads, 0, st>>>(
                units_raw.p, dnu.p, key.p, bucket.p, t.units.p);
            BT_LAUNCH("unit_scatter");
        }
    }
    // the build's one closing control read: statistics, root box, root b, input check
    unsigned long long hstat[4];
    double hb[8];
    int hbad = 0;
    int32_t rb = 0;
    long long nu = 0;
    if (t.root_is_leaf)
        read_back({{dstat.p, hstat, 4 * sizeof(unsigned long long)}, {dbox.p, hb, 7 * sizeof(double)},
                   {dflags.p, &hbad, sizeof(int)}, {dnu.p, &nu, sizeof(long long)}});
    else
        read_back({{dstat.p, hstat, 4 * sizeof(unsigned long long)}, {dbox.p, hb, 7 * sizeof(double)},
                   {dflags.p, &hbad, sizeof(int)}, {&t.nodes.p[0].b, &rb, sizeof(int32_t)},
                   {dnu.p, &nu, sizeof(long long)}});
    t.n_units = nu;
    if (hbad) throw Error(BT_ERR_INPUT, "bt_build: non-finite coordinate or |coordinate| > 1e150");
    for (int l = 0; l < 3; l++) {
        t.box_lo[l] = hb[l];
        t.box_hi[l] = hb[3 + l];
    }
    t.M = hb[6];
    t.root_b = rb;
    t.halvings = (int64_t)hstat[0];
    t.max_leaf = (int64_t)hstat[1];
    t.overfull = (int64_t)hstat[2];
}

}  // namespace bt
