/*
 * btree.h -- C ABI of the B200-native b-tree exact close-neighbor search.
 *
 * The method is the b-tree of Cavelan, Cabezon, Korndorfer, Ciorba,
 * "Finding Neighbors in a Forest: A b-tree for Smoothed Particle Hydrodynamics
 * Simulations" (arXiv 1910.02639).  P:n below is line n of that paper's text
 * with the section / equation / algorithm it falls in.
 *
 * Result computed (the plain definition, BASELINE.json north_star):
 *   N(i) = { j in [0,n), j != i :
 *            ((dx*dx + dy*dy) + dz*dz) < (2 h_i) * (2 h_i) }
 *   dx = x_i - x_j (likewise y, z), IEEE-754 binary64, round-to-nearest-even,
 *   each operation rounded separately (no FMA), left to right.  This is the
 *   paper's "all particles that are within the 2h radius" (Sec. III-B,
 *   P:266-280) with the gather radius of the query (Alg. 2 uses h_p),
 *   strict inequality (reading R1 in DESIGN.md) and self excluded (R12).
 *   The set is a function of the inputs alone: it does not depend on the tree,
 *   bucket_size, max_empty or alpha.
 *
 * Conventions for every entry point
 *   - Device pointers are CUDA global-memory pointers of the current device
 *     (e.g. torch CUDA tensors' data_ptr()); host pointers are plain memory.
 *   - All work is enqueued on the calling thread's stream (bt_set_stream;
 *     default: the per-thread default stream) and the call returns after the
 *     work has completed (it synchronises that stream).
 *   - Inputs and outputs are in CALLER order: particle i is row i of pos/h.
 *   - Return codes: BT_OK or one of bt_status; constructors return NULL on
 *     failure.  The message of the last failure on this thread is in
 *     bt_last_error(), its code in bt_last_status().  No C++ exception crosses
 *     this boundary.
 *   - A bt_tree may be used by one thread at a time (it owns scratch memory).
 */
#ifndef BTREE_H
#define BTREE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bt_tree bt_tree; /* opaque, library-owned */

typedef enum bt_status {
    BT_OK = 0,
    BT_ERR_ARG = 1,      /* invalid argument (NULL pointer, range, size)        */
    BT_ERR_INPUT = 2,    /* invalid data (non-finite or |coordinate| > 1e150,
                            h not finite, h <= 0 or h > 1e150)                   */
    BT_ERR_CAPACITY = 3, /* neighbor output does not fit the given capacity      */
    BT_ERR_CUDA = 4,     /* CUDA runtime / launch failure                        */
    BT_ERR_OOM = 5       /* device memory exhausted                              */
} bt_status;

/*
 * bt_build -- BuildTree (Alg. 1; Eq. 1-4) on the device.
 *
 *   pos          DEVICE, n*3 fp64, AoS x,y,z per particle, caller-owned,
 *                read-only; finite with |coordinate| <= 1e150.  The tree keeps
 *                its own copy (records in depth-first leaf order, Sec. IV-E
 *                P:491), so pos may be freed after the call.
 *   n            0 <= n <= 2^31 - 1.  n == 0 gives a valid empty tree.
 *   bucket_size  s >= 1: maximum particles per leaf (Table I).
 *   max_empty    beta in (0, 1]: a node's branching factor b is halved while
 *                the ratio r of sub-cells holding <= alpha*s particles is
 *                >= beta and b > 2 (Eq. 4 + Step 3; readings R3, R4,
 *                R7).  alpha = 0.5 (Table IV; reading R10).
 *
 * The root box is the data's bounding box, each side expanded by
 * max(1e-9 * extent, 1e-12) (reading R9).  Nodes at depth 64 become leaves
 * even when they hold more than s particles (coincident points, R14).
 * Returns NULL on failure (BT_ERR_ARG / BT_ERR_INPUT / BT_ERR_CUDA / BT_ERR_OOM).
 */
bt_tree *bt_build(const double *pos, int64_t n, int32_t bucket_size, double max_empty);

/* bt_build with alpha in [0, 1] (Table I) and the depth cap (>= 0). */
bt_tree *bt_build_ex(const double *pos, int64_t n, int32_t bucket_size, double max_empty,
                     double alpha, int32_t depth_cap);

/*
 * bt_build_policy -- bt_build_ex with a subdivision policy:
 *   BT_POLICY_BTREE   the paper's adaptive b (Eq. 1 + the Eq. 4 halving loop);
 *   BT_POLICY_OCTREE  the classical octree the paper compares against (Sec. II,
 *                     P:98-103; Table II): b = 2 at every node, no ratio test
 *                     (max_empty and alpha are ignored);
 *   BT_POLICY_BTREE_2D  the b-tree with k = 2 (the paper is k-generic, Table I
 *                     P:140; reading R23): Eq. 1 with b^2 s >= n_i, b^2
 *                     sub-cells per node (x and y divided, z one slab), the
 *                     Eq. 4 ratio over the b^2 sub-cells;
 *   BT_POLICY_QUADTREE  b = 2 with k = 2, no ratio test.
 * pos stays [n,3]; the k = 2 trees suit planar (2-D) particle sets and are
 * valid for any input.  The neighbor sets found through any of these trees
 * are identical.
 */
enum { BT_POLICY_BTREE = 0, BT_POLICY_OCTREE = 1, BT_POLICY_BTREE_2D = 2, BT_POLICY_QUADTREE = 3 };
bt_tree *bt_build_policy(const double *pos, int64_t n, int32_t bucket_size, double max_empty,
                         double alpha, int32_t depth_cap, int32_t policy);

/*
 * bt_find_neighbors -- FindNeighbors (Alg. 2; Eq. 5)
 * for every particle of the tree, count-then-fill CSR output.
 *
 *   t        tree from bt_build (the particles whose neighbors are searched
 *            and the candidate set are the same n particles).
 *   h        DEVICE, n fp64 smoothing lengths in caller order, finite, > 0.
 *   ngmax    >= 1; nbr_idx has capacity n * ngmax entries.  A capacity, not a
 *            truncation: counts are exact and never clamped (reading R17).
 *   counts   DEVICE out, n int32: counts[i] = |N(i)|.
 *   offsets  DEVICE out, n+1 int64: exclusive scan of counts, offsets[n] = total.
 *   nbr_idx  DEVICE out, int32, capacity n*ngmax, or NULL for a count-only call.
 *            Row i = nbr_idx[offsets[i] .. offsets[i+1]) holds the caller
 *            indices j of N(i) in unspecified order.
 *
 * Returns BT_OK; BT_ERR_ARG (NULL t/h/counts/offsets with n > 0, ngmax < 1);
 * BT_ERR_INPUT (bad h; outputs undefined); BT_ERR_CAPACITY when
 * offsets[n] > n*ngmax: counts and offsets are valid, nbr_idx is untouched,
 * and the caller may retry with bt_fill_neighbors and a larger buffer.
 */
int bt_find_neighbors(const bt_tree *t, const double *h, int32_t ngmax, int32_t *counts,
                      int64_t *offsets, int32_t *nbr_idx);

/*
 * bt_fill_neighbors -- the fill pass alone, using offsets from a previous
 * bt_find_neighbors call on the same tree and the same h (e.g. count-only,
 * then an exactly sized buffer).  capacity = number of int32 slots of nbr_idx;
 * BT_ERR_CAPACITY if offsets[n] > capacity (nothing written); BT_ERR_ARG if
 * offsets are not the exclusive scan of this tree's counts for this h and
 * partition (checked exactly when the count pass is redone, else by a
 * checksum of the recorded counts; nothing written).
 */
int bt_fill_neighbors(const bt_tree *t, const double *h, const int64_t *offsets,
                      int32_t *nbr_idx, int64_t capacity);

/*
 * bt_density -- SPH density with the neighbor search fused in (SURVEY 8(f)
 * row 3: the use the paper builds the lists for, Sec. I, Sec. IV-H
 * P:540-549), without materialising the CSR.  Reading R21 (the
 * paper does not fix a kernel): the M4 cubic spline of compact support 2h,
 *   rho_i = ( m_i w(0) + sum_{j in N(i)} m_j w(r_ij / h_i) ) / (pi h_i^3),
 *   w(q) = 1 - 1.5 q^2 + 0.75 q^3 (q < 1),  0.25 (2 - q)^3 (1 <= q < 2),
 * with N(i) exactly the neighbor set of bt_find_neighbors (the same walk and
 * exact predicate).  The pair distances r_ij are evaluated in fp32 from the
 * unit-relative coordinates of lemma L4 and the sum of each 128-candidate
 * block in fp32, blocks accumulated in fp64: relative error <= 1e-4 of rho
 * (DESIGN.md section 11c).
 *   h    DEVICE, n fp64, caller order, finite, > 0 (as bt_find_neighbors)
 *   mass DEVICE, n fp64, caller order, finite
 *   rho  DEVICE out, n fp64, caller order
 * Errors: BT_ERR_ARG (NULL tree / pointers), BT_ERR_INPUT (bad h or mass),
 * BT_ERR_CUDA / BT_ERR_OOM.  Enqueued on the thread's stream; returns after
 * completion.  Does not touch the masks a previous count pass recorded
 * (a later bt_fill_neighbors recomputes them).
 */
int bt_density(const bt_tree *t, const double *h, const double *mass, double *rho);

/*
 * bt_find_neighbors_sym -- the symmetric criterion (the
 * paper's Alg. 2 uses the query's h only; the open question of
 * SPEC S:273; reading R22 in DESIGN.md): j != i is a neighbor of i iff
 *   ((dx*dx + dy*dy) + dz*dz) < (2 max(h_i, h_j)) * (2 max(h_i, h_j))
 * in fp64 (no FMA), dx = x_i - x_j.  Equivalently N_sym(i) = N(i) u
 * {j : i in N(j)} with N the gather sets of bt_find_neighbors.  It is
 * searched from the query side in one walk: the descent and culls use
 * max(R'_i, R'(h_max)) with h_max the largest h of each node / leaf, and
 * every pair is tested against both thresholds (DESIGN.md lemma L4s).  The
 * relation is symmetric.  Arguments, layouts, ownership, synchrony, row
 * order (unspecified), the count-only call (nbr_idx NULL), partitions
 * (bt_set_partition) and the errors are those of bt_find_neighbors
 * (capacity n*ngmax; BT_ERR_CAPACITY leaves counts and offsets valid and
 * nbr_idx untouched).  Uses internal device memory of (leaves + nodes) fp64
 * besides the gather pass's.
 */
int bt_find_neighbors_sym(const bt_tree *t, const double *h, int32_t ngmax, int32_t *counts,
                          int64_t *offsets, int32_t *nbr_idx);

/*
 * bt_fill_neighbors_sym -- the fill of bt_find_neighbors_sym alone, with the
 * offsets of a previous symmetric count on the same tree and h (the count
 * pass is reused when nothing ran in between, else redone).  capacity =
 * int32 slots of nbr_idx; BT_ERR_CAPACITY if offsets[n] > capacity;
 * BT_ERR_ARG if offsets are not the scan of this tree's symmetric counts for
 * this h and partition.
 */
int bt_fill_neighbors_sym(const bt_tree *t, const double *h, const int64_t *offsets,
                          int32_t *nbr_idx, int64_t capacity);

/*
 * bt_set_partition -- restrict this tree's later searches to part `part` of
 * `nparts` (the replicated-tree multi-GPU variant of SURVEY 8(e): every rank
 * builds the same tree from the same positions and searches only its share).
 * The parts are contiguous ranges of the Morton-ordered work units (units
 * [U*part/nparts, U*(part+1)/nparts) of U), i.e. spatially compact sets of
 * whole leaves; every particle belongs to exactly one part.  Afterwards
 * bt_find_neighbors / bt_fill_neighbors return counts[i] = |N(i)| and row i
 * for the particles of the part and counts 0 (empty rows) for all others, so
 * the CSR sizes to the part; bt_density writes rho only for the part's
 * particles; bt_find_neighbors_sym the part's symmetric rows.  nparts = 1
 * restores the whole tree.  BT_ERR_ARG for
 * nparts < 1 or part outside [0, nparts).  No device work.
 */
int bt_set_partition(bt_tree *t, int32_t part, int32_t nparts);

/*
 * bt_set_tree_order -- the index space of this tree's later searches.  The
 * paper's first walk optimisation is that "particles are reordered in memory
 * along this curve" (the depth-first leaf order of the tree walk); a
 * caller that keeps its particles in that order works in tree positions
 * k = 0 .. n-1 (particle perm[k] of bt_tree_order).  With on != 0, every
 * per-particle array of bt_find_neighbors(_sym), bt_fill_neighbors(_sym) and
 * bt_density is indexed by tree position: h[k], mass[k], counts[k], row k of
 * offsets / nbr_idx and rho[k] belong to particle perm[k], and the neighbor
 * indices written to nbr_idx are tree positions.  The neighbor sets are
 * those of the default (caller-order) space mapped through perm: row k holds
 * {perm^-1(j) : j in N(perm[k])}.  Equivalently, the result equals the
 * default-space search of the reordered particle set pos[perm] (whose tree
 * has the identity permutation).  on = 0 restores caller order (the
 * default).  Rows of consecutive tree positions are adjacent in nbr_idx, so
 * the fill pass writes each work unit's rows as one contiguous range.
 * Invalidates the recorded count pass.  No device work.  BT_ERR_ARG for a
 * NULL tree.
 */
int bt_set_tree_order(bt_tree *t, int on);

/*
 * bt_reorder -- gather a caller-order array into tree order:
 *   dst[k * ncomp + c] = src[perm[k] * ncomp + c],  k < n, c < ncomp,
 * perm = bt_tree_order's (e.g. h or masses for bt_set_tree_order, or
 * positions with ncomp = 3).  src, dst: DEVICE fp64, n * ncomp each, caller
 * owned, must not overlap.  ncomp in [1, 16].  Values are copied bit for bit
 * (no validation).  BT_ERR_ARG for a NULL tree / pointers or ncomp outside
 * [1, 16].  Enqueued on the thread's stream; returns after completion.
 */
int bt_reorder(const bt_tree *t, const double *src, int32_t ncomp, double *dst);

/* Frees all tree-owned device memory (into this thread's block cache).  NULL-safe. */
void bt_free(bt_tree *t);

/*
 * Device memory comes from a per-thread block cache over cudaMalloc: blocks
 * freed by bt_free or by internal scratch are reused by later calls of the
 * same thread (repeated builds cost no driver allocation).  This returns the
 * cached blocks of the calling thread to the driver.
 */
int bt_release_cache(void);

/*
 * bt_search_host -- end-to-end convenience call on HOST buffers: copies pos
 * and h to the device, builds, counts, scans and fills, and copies counts,
 * offsets and the neighbor lists back.  Host buffers should be pinned
 * (cudaHostAlloc / torch pin_memory) for full PCIe bandwidth.
 *   pos_h [n*3] fp64, h_h [n] fp64, counts_h [n] int32, offsets_h [n+1] int64,
 *   nbr_h [capacity] int32.  BT_ERR_CAPACITY if the total exceeds capacity
 *   (counts_h and offsets_h are then valid, nbr_h untouched).
 */
int bt_search_host(const double *pos_h, const double *h_h, int64_t n, int32_t bucket_size,
                   double max_empty, int32_t *counts_h, int64_t *offsets_h, int32_t *nbr_h,
                   int64_t capacity);

/* Stream for this thread's subsequent calls (a cudaStream_t; NULL = default). */
int bt_set_stream(void *cuda_stream);

/*
 * Validation knob (thread-local): on != 0 sends every candidate pair to the
 * fp64 predicate itself instead of deciding the certain cases with the fp32
 * pre-test of lemma L4.  Results are identical by
 * construction; tests use it to check that, bench-style runs to measure it.
 */
int bt_set_exact_only(int on);

const char *bt_last_error(void);
int bt_last_status(void);

typedef struct bt_stats {
    int64_t n;
    int64_t nodes;        /* internal nodes                                   */
    int64_t leaves;
    int64_t halvings;     /* total b-halving rounds over all nodes (Eq. 4)    */
    int64_t overfull;     /* leaves with more than s particles (depth cap)    */
    int64_t max_leaf;
    int32_t depth;        /* leaf depth maximum; a root leaf has depth 0      */
    int32_t root_b;       /* accepted branching factor of the root (0: leaf)  */
    int64_t units;        /* walk work units (a leaf, a 64-query part of one, or two small leaves) */
    double box_lo[3], box_hi[3];
    /* last bt_find_neighbors on this tree */
    int64_t total_pairs;
    int64_t max_count;
    int64_t staged;       /* candidate records staged by the count pass       */
    int64_t tests;        /* pair tests issued by the count pass              */
    int64_t exact_tests;  /* pairs decided by the fp64 predicate itself       */
    int64_t loaded;       /* particle records read by the staging (before the cull) */
    int64_t mask_words;   /* 64-bit neighbor mask words allocated for the fill pass */
    int64_t cand_slots;   /* candidate arena slots allocated                     */
    int64_t list_entries; /* candidate-leaf list entries allocated by the descent */
    int64_t big_units;    /* units redone by the global-frontier descent pass    */
    int64_t rows_over_ngmax; /* rows of the last count with more than its ngmax neighbors
                                (SPH callers sizing fixed-stride tables; counts are never clamped) */
    int64_t mask_words_nonzero; /* recorded mask words holding at least one neighbor (the fill's work) */
} bt_stats;

int bt_tree_stats(const bt_tree *t, bt_stats *out);

/*
 * bt_tree_order -- export the tree (DEVICE outputs, any may be NULL):
 *   perm[n]         caller index of the particle at each tree-order position
 *                   (depth-first leaf order, children in ascending sub-cell id j,
 *                   ascending caller index inside a leaf: Sec. IV-E);
 *   leaf_begin[L]   first tree-order position of each leaf (depth-first order);
 *   leaf_count[L]   particles in the leaf;
 *   leaf_depth[L]   depth of the leaf.
 * L = bt_stats.leaves.
 */
int bt_tree_order(const bt_tree *t, int32_t *perm, int64_t *leaf_begin, int32_t *leaf_count,
                  int32_t *leaf_depth);

/*
 * Profiling: when enabled, every kernel phase is bracketed with CUDA events on
 * the library's stream and its time accumulated (ms).  bt_profile_get fills
 * names/values; returns the number of entries.  Launch counts are always kept.
 */
int bt_profile_enable(int on);
int bt_profile_reset(void);
int bt_profile_get(int max_entries, const char **names, double *ms, int64_t *launches);

#ifdef __cplusplus
}
#endif

#endif /* BTREE_H */
