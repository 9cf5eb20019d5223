/*
 * btree_oracle.c -- CPU ORACLE FOR THE b-tree EXACT CLOSE-NEIGHBOR SEARCH.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1910_02639_b200/) never links, imports or calls it,
 * and it shares no code, header, table or constant generator with the CUDA
 * library.  It is deliberately plain and slow: recursive BuildTree (Alg. 1)
 * and recursive FindNeighbors (Alg. 2) written in the paper's order and
 * notation, plus an O(n^2) brute force that implements the plain definition.
 *
 * Citations: P:n = line n of the paper text (PAPER.md, arXiv 1910.02639),
 * with the section / equation / algorithm it falls in.  Readings of the paper
 * where it is silent or garbled are numbered R1..R23 in DESIGN.md section 3.
 *
 * Build flags (see __graft_entry__.build): gcc -O2 -std=c11 -fPIC -shared
 * -ffp-contract=off -fno-fast-math -fopenmp.  x86-64 SSE2 fp64, no FMA, no
 * x87, no FTZ: every fp64 operation below is one IEEE-754 binary64 operation
 * in round-to-nearest-even, in the order written.
 *
 * Pinned by tests/test_oracle_pins.py (worked examples of Eq. 2/3, Eq. 1 and
 * Eq. 4 closed forms, Fig. 1 ranges, lattice neighbor counts, boundary
 * convention, brute force vs scipy cKDTree, structural invariants; the k = 2
 * policies, the symmetric criterion and the density sum by their own closed
 * forms and cross-checks).  Tree shapes at scale are "parity unpinned"
 * beyond those invariants.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* Eq. 1 (Sec. III-A Step 1): b = ceil((n/s)^(1/k)), k = 3.  */
/* Reading R6: the smallest integer b >= 2 with b^3 * s >= n, computed  */
/* with integers (pow() lands just below integers).                    */
/* ------------------------------------------------------------------ */
int orc_branching_factor(int64_t n, int64_t s)
{
    int64_t m = (n + s - 1) / s; /* ceil(n/s): b^3*s >= n  <=>  b^3 >= ceil(n/s) */
    int64_t b = 2;
    while (b * b * b < m)
        b++;
    return (int)b;
}

/* Eq. 1 for k dimensions (the paper is k-generic, Table I): the    */
/* smallest integer b >= 2 with b^k * s >= n, k in {2, 3} (R23).          */
int orc_branching_factor_k(int64_t n, int64_t s, int k)
{
    int64_t m = (n + s - 1) / s;
    int64_t b = 2;
    while ((k == 3 ? b * b * b : b * b) < m)
        b++;
    return (int)b;
}

/* ------------------------------------------------------------------ */
/* Eq. 2 (Sec. III-A Step 2):                               */
/*   x'_l = floor( (x_l - x_{l,min}) / (x_{l,max} - x_{l,min}) * b )   */
/* Reading R8: clamp to [0, b-1] (upper-face particles); a NaN (only   */
/* possible as 0/0 on a zero-extent box) maps to 0, which keeps the map */
/* monotone non-decreasing in x (lemma L2).                 */
/* ------------------------------------------------------------------ */
int orc_cell_coord(double x, double lo, double hi, int b)
{
    double q = ((x - lo) / (hi - lo)) * (double)b;
    double f = floor(q);
    if (!(f >= 0.0))
        return 0;
    if (f > (double)(b - 1))
        return b - 1;
    return (int)f;
}

/* Eq. 3: j = x'_1 + x'_2 W + x'_3 W^2, with W = b (R5). */
int64_t orc_cell_id(int c1, int c2, int c3, int b)
{
    return (int64_t)c1 + (int64_t)c2 * b + (int64_t)c3 * b * b;
}

/* Eq. 4 (Sec. III-A Step 3): r = #{j : n_j <= alpha*s} / b^k. */
/* Reading R4: the Iverson bracket with <=, empty cells count.           */
double orc_ratio(const int64_t *counts, int64_t ncells, double alpha, int64_t s)
{
    int64_t u = 0;
    for (int64_t j = 0; j < ncells; j++)
        if ((double)counts[j] <= alpha * (double)s)
            u++;
    return (double)u / (double)ncells;
}

/* Eq. 5 (Sec. III-B): inclusive index range of the sub-cells */
/* that can hold a particle within distance R of x along one axis.      */
/* Reading R11: clamped to [0, b-1]; R is the widened radius R' below.  */
void orc_range(double x, double R, double lo, double hi, int b, int *rmin, int *rmax)
{
    *rmin = orc_cell_coord(x - R, lo, hi, b);
    *rmax = orc_cell_coord(x + R, lo, hi, b);
}

/* Pair predicate ("less than 2h_p"; Alg. 2), reading R1/R2  */
/* fixed by BASELINE.json: ((dx*dx + dy*dy) + dz*dz) < (2h)*(2h), fp64,  */
/* left to right, no FMA (compiled with -ffp-contract=off).             */
static int orc_pair(const double *xi, const double *xj, double T)
{
    double dx = xi[0] - xj[0];
    double dy = xi[1] - xj[1];
    double dz = xi[2] - xj[2];
    double d2 = (dx * dx + dy * dy) + dz * dz;
    return d2 < T;
}

/* Root box (SPEC core-model compute_root_box; reading R9): exact per-axis */
/* min/max, each side expanded by max(1e-9 * extent, 1e-12).              */
void orc_root_box(const double *pos, int64_t n, double *lo, double *hi)
{
    for (int l = 0; l < 3; l++) {
        double mn = pos[l], mx = pos[l];
        for (int64_t i = 1; i < n; i++) {
            double v = pos[3 * i + l];
            if (v < mn) mn = v;
            if (v > mx) mx = v;
        }
        double pad = 1e-9 * (mx - mn);
        if (pad < 1e-12)
            pad = 1e-12;
        lo[l] = mn - pad;
        hi[l] = mx + pad;
    }
}

/* ------------------------------------------------------------------ */
/* Tree (Alg. 1).  Children are stored sparsely: only the   */
/* non-empty sub-cells, in ascending j ("only non-empty cells need */
/* to be stored").                                                     */
/* ------------------------------------------------------------------ */
typedef struct orc_node {
    double lo[3], hi[3];
    int b;          /* accepted branching factor (internal nodes) */
    int bz;         /* sub-cells along z: b, or 1 for k = 2 */
    int depth;
    int halvings;   /* redistribution rounds that halved b */
    int is_leaf;
    int overfull;   /* leaf with more than s particles (depth cap, R14) */
    int64_t n;      /* particles under this node */
    int32_t *idx;   /* leaf: particle indices, ascending original index */
    int64_t nchild;
    int64_t *child_j;          /* ascending sub-cell ids of non-empty cells */
    struct orc_node **child;
} orc_node;

typedef struct {
    int64_t n;
    int32_t s;
    double beta, alpha;
    int32_t depth_cap;
    int octree; /* FixedOctree policy: b = 2, no ratio loop (Sec. II) */
    int k;      /* dimensions subdivided: 3, or 2 (x, y only; z is one slab) (R23) */
    double box_lo[3], box_hi[3];
    double M;       /* max |root box coordinate|, for the radius margin */
    orc_node *root; /* NULL iff n == 0 */
    /* statistics */
    int64_t nodes, leaves, halvings, overfull;
    int depth, root_b;
    int64_t max_leaf;
} orc_tree;

typedef struct {
    int64_t n, nodes, leaves, halvings, overfull, max_leaf;
    int32_t depth, root_b;
} orc_stats;

static orc_node *new_leaf(orc_tree *t, const double *lo, const double *hi,
                          int32_t *idx, int64_t n, int depth)
{
    orc_node *nd = (orc_node *)calloc(1, sizeof(orc_node));
    memcpy(nd->lo, lo, sizeof(nd->lo));
    memcpy(nd->hi, hi, sizeof(nd->hi));
    nd->is_leaf = 1;
    nd->depth = depth;
    nd->n = n;
    nd->idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    memcpy(nd->idx, idx, sizeof(int32_t) * (size_t)n);
    nd->overfull = n > t->s;
    t->leaves++;
    t->overfull += nd->overfull;
    if (depth > t->depth) t->depth = depth;
    if (n > t->max_leaf) t->max_leaf = n;
    return nd;
}

/* BuildTree(n, i), Alg. 1 P:175-202.  idx holds the particles of cell i */
/* in ascending original index.                                          */
static orc_node *build_tree(orc_tree *t, const double *pos, const double *lo,
                            const double *hi, int32_t *idx, int64_t n, int depth)
{
    /* A cell with n <= s is a leaf; so is a cell at the depth cap */
    /* (reading R14: Alg. 1 would recurse forever on s+1 equal points).   */
    if (n <= t->s || depth >= t->depth_cap)
        return new_leaf(t, lo, hi, idx, n, depth);

    orc_node *nd = (orc_node *)calloc(1, sizeof(orc_node));
    memcpy(nd->lo, lo, sizeof(nd->lo));
    memcpy(nd->hi, hi, sizeof(nd->hi));
    nd->depth = depth;
    nd->n = n;
    t->nodes++;

    /* Step 1: branching factor, Eq. 1 (computed once, then only halved: R6). */
    /* The octree policy fixes b = 2 and skips Step 3.                       */
    int b = t->octree ? 2 : orc_branching_factor_k(n, t->s, t->k);
    int64_t *cell = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *cnt = NULL;
    int64_t B = 0;
    for (;;) {
        /* Step 2: create b^k sub-cells and distribute the particles (Eq. 2, 3). */
        /* k = 2: the z axis is not divided (one slab, b_z = 1, so c3 = 0).      */
        int bz = t->k == 3 ? b : 1;
        B = (int64_t)b * b * bz;
        free(cnt);
        cnt = (int64_t *)calloc((size_t)B, sizeof(int64_t));
        for (int64_t p = 0; p < n; p++) {
            const double *x = pos + 3 * (int64_t)idx[p];
            int c1 = orc_cell_coord(x[0], lo[0], hi[0], b);
            int c2 = orc_cell_coord(x[1], lo[1], hi[1], b);
            int c3 = orc_cell_coord(x[2], lo[2], hi[2], bz);
            int64_t j = orc_cell_id(c1, c2, c3, b);
            cell[p] = j;
            cnt[j]++; /* "Update n_j" */
        }
        /* Step 3: distribution ratio, Eq. 4; halve while r >= beta (R3, R7). */
        if (t->octree)
            break;
        double r = orc_ratio(cnt, B, t->alpha, t->s);
        if (r >= t->beta && b > 2) {
            b = b / 2;
            if (b < 2) b = 2;
            nd->halvings++;
        } else {
            break;
        }
    }
    nd->b = b;
    nd->bz = t->k == 3 ? b : 1;
    t->halvings += nd->halvings;

    /* Stable distribution into per-cell lists (ascending original index). */
    int64_t *start = (int64_t *)malloc(sizeof(int64_t) * (size_t)(B + 1));
    start[0] = 0;
    int64_t nonempty = 0;
    for (int64_t j = 0; j < B; j++) {
        start[j + 1] = start[j] + cnt[j];
        if (cnt[j] > 0) nonempty++;
    }
    int32_t *sorted = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)B);
    memcpy(fill, start, sizeof(int64_t) * (size_t)B);
    for (int64_t p = 0; p < n; p++)
        sorted[fill[cell[p]]++] = idx[p];
    free(fill);
    free(cell);

    /* For each non-empty sub-cell j (ascending): BuildTree if n_j > s, else */
    /* a leaf (Alg. 1).  Child box = equal 1/b slice of the cell.  */
    nd->nchild = nonempty;
    nd->child_j = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nonempty > 0 ? nonempty : 1));
    nd->child = (orc_node **)malloc(sizeof(orc_node *) * (size_t)(nonempty > 0 ? nonempty : 1));
    int64_t k = 0;
    for (int64_t j = 0; j < B; j++) {
        if (cnt[j] == 0)
            continue;
        int c[3];
        c[0] = (int)(j % b);
        c[1] = (int)((j / b) % b);
        c[2] = (int)(j / ((int64_t)b * b));
        double clo[3], chi[3];
        for (int l = 0; l < 3; l++) {
            double bl = (l == 2 && t->k == 2) ? 1.0 : (double)b; /* b_z = 1 for k = 2 */
            clo[l] = lo[l] + ((double)c[l] * (hi[l] - lo[l])) / bl;
            chi[l] = lo[l] + ((double)(c[l] + 1) * (hi[l] - lo[l])) / bl;
        }
        nd->child_j[k] = j;
        nd->child[k] = build_tree(t, pos, clo, chi, sorted + start[j], cnt[j], depth + 1);
        k++;
    }
    free(sorted);
    free(start);
    free(cnt);
    return nd;
}

orc_tree *orc_build_policy(const double *pos, int64_t n, int32_t s, double beta,
                           double alpha, int32_t depth_cap, int policy);

orc_tree *orc_build(const double *pos, int64_t n, int32_t s, double beta,
                    double alpha, int32_t depth_cap)
{
    return orc_build_policy(pos, n, s, beta, alpha, depth_cap, 0);
}

/* policy: 0 b-tree (k = 3), 1 octree (b = 2, k = 3), 2 b-tree with k = 2, */
/* 3 quadtree (b = 2, k = 2).                                             */
orc_tree *orc_build_policy(const double *pos, int64_t n, int32_t s, double beta,
                           double alpha, int32_t depth_cap, int policy)
{
    if (n < 0 || s < 1 || !(beta > 0.0 && beta <= 1.0) || depth_cap < 0 || policy < 0 || policy > 3)
        return NULL;
    orc_tree *t = (orc_tree *)calloc(1, sizeof(orc_tree));
    t->n = n;
    t->s = s;
    t->beta = beta;
    t->alpha = alpha;
    t->depth_cap = depth_cap;
    t->octree = policy == 1 || policy == 3;
    t->k = policy >= 2 ? 2 : 3;
    if (n == 0)
        return t;
    orc_root_box(pos, n, t->box_lo, t->box_hi);
    double M = 0.0;
    for (int l = 0; l < 3; l++) {
        if (fabs(t->box_lo[l]) > M) M = fabs(t->box_lo[l]);
        if (fabs(t->box_hi[l]) > M) M = fabs(t->box_hi[l]);
    }
    t->M = M;
    int32_t *idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    for (int64_t i = 0; i < n; i++)
        idx[i] = (int32_t)i;
    t->root = build_tree(t, pos, t->box_lo, t->box_hi, idx, n, 0);
    t->root_b = t->root->is_leaf ? 0 : t->root->b;
    free(idx);
    return t;
}

static void free_node(orc_node *nd)
{
    if (!nd)
        return;
    for (int64_t k = 0; k < nd->nchild; k++)
        free_node(nd->child[k]);
    free(nd->child);
    free(nd->child_j);
    free(nd->idx);
    free(nd);
}

void orc_free(orc_tree *t)
{
    if (!t)
        return;
    free_node(t->root);
    free(t);
}

int orc_get_stats(const orc_tree *t, orc_stats *out)
{
    out->n = t->n;
    out->nodes = t->nodes;
    out->leaves = t->leaves;
    out->halvings = t->halvings;
    out->overfull = t->overfull;
    out->max_leaf = t->max_leaf;
    out->depth = t->depth;
    out->root_b = t->root_b;
    return 0;
}

void orc_get_box(const orc_tree *t, double *lo, double *hi)
{
    memcpy(lo, t->box_lo, sizeof(t->box_lo));
    memcpy(hi, t->box_hi, sizeof(t->box_hi));
}

/* Depth-first leaf order, children in ascending j: the order in which the */
/* paper reorders particles (Sec. IV-E).                            */
static void dfs_leaves(const orc_node *nd, int32_t *perm, int64_t *pos,
                       int64_t *lbegin, int32_t *lcount, int32_t *ldepth,
                       int64_t *nleaf)
{
    if (nd->is_leaf) {
        if (lbegin) lbegin[*nleaf] = *pos;
        if (lcount) lcount[*nleaf] = (int32_t)nd->n;
        if (ldepth) ldepth[*nleaf] = nd->depth;
        (*nleaf)++;
        if (perm) memcpy(perm + *pos, nd->idx, sizeof(int32_t) * (size_t)nd->n);
        *pos += nd->n;
        return;
    }
    for (int64_t k = 0; k < nd->nchild; k++)
        dfs_leaves(nd->child[k], perm, pos, lbegin, lcount, ldepth, nleaf);
}

/* perm[n]: particle indices in depth-first leaf order; leaves: begin/count/ */
/* depth per leaf in the same order (any pointer may be NULL).  Returns the  */
/* number of leaves.                                                        */
int64_t orc_get_order(const orc_tree *t, int32_t *perm, int64_t *lbegin,
                      int32_t *lcount, int32_t *ldepth)
{
    int64_t p = 0, nl = 0;
    if (t->root)
        dfs_leaves(t->root, perm, &p, lbegin, lcount, ldepth, &nl);
    return nl;
}

/* ------------------------------------------------------------------ */
/* FindNeighbors(p, h_p, i), Alg. 2 P:282-303.                          */
/* The range radius is widened from 2h to                              */
/*   R' = 2h (1 + 2^-40) + 2^-50 M   (reading R11, lemma L1/L2)         */
/* so that rounding in Eq. 5 never drops a neighbor; the leaf test is   */
/* the exact predicate.                                                 */
/* ------------------------------------------------------------------ */
typedef struct {
    int32_t *buf; /* NULL: count only */
    int64_t cap;
    int64_t len;
} orc_row;

static void leaf_test(const orc_node *leaf, const double *pos, int64_t p,
                      double T, orc_row *row)
{
    const double *xp = pos + 3 * p;
    for (int64_t k = 0; k < leaf->n; k++) {
        int64_t q = leaf->idx[k];
        if (q == p)
            continue; /* self is not its own neighbor (R12) */
        if (orc_pair(xp, pos + 3 * q, T)) {
            if (row->buf && row->len < row->cap)
                row->buf[row->len] = (int32_t)q;
            row->len++; /* "Add q to NeighborsOf(p)" */
        }
    }
}

static void find_neighbors(const orc_node *nd, const double *pos, int64_t p,
                           double T, double Rp, orc_row *row)
{
    if (nd->is_leaf) { /* only the root can be reached here as a leaf */
        leaf_test(nd, pos, p, T, row);
        return;
    }
    const double *x = pos + 3 * p;
    int r[3][2];
    for (int l = 0; l < 3; l++) /* Eq. 5 per axis; k = 2: one z slab (b_z = 1) */
        orc_range(x[l], Rp, nd->lo[l], nd->hi[l], (l == 2 && nd->bz == 1) ? 1 : nd->b, &r[l][0], &r[l][1]);
    int64_t lo_k = 0;
    for (int c3 = r[2][0]; c3 <= r[2][1]; c3++)
        for (int c2 = r[1][0]; c2 <= r[1][1]; c2++)
            for (int c1 = r[0][0]; c1 <= r[0][1]; c1++) {
                int64_t j = orc_cell_id(c1, c2, c3, nd->b);
                /* Locate sub-cell j among the stored (non-empty) children. */
                int64_t a = lo_k, z = nd->nchild;
                while (a < z) {
                    int64_t m = a + (z - a) / 2;
                    if (nd->child_j[m] < j) a = m + 1; else z = m;
                }
                lo_k = a; /* j is increasing in this loop order */
                if (a >= nd->nchild || nd->child_j[a] != j)
                    continue; /* empty sub-cell */
                const orc_node *ch = nd->child[a];
                if (ch->is_leaf) /* n_j <= s (or depth-capped): test each q */
                    leaf_test(ch, pos, p, T, row);
                else /* n_j > s: recurse */
                    find_neighbors(ch, pos, p, T, Rp, row);
            }
}

static void one_row(const orc_tree *t, const double *pos, const double *h,
                    int64_t p, orc_row *row)
{
    double tt = 2.0 * h[p];
    double T = tt * tt;
    double Rp = tt * (1.0 + 0x1p-40) + 0x1p-50 * t->M;
    if (t->root)
        find_neighbors(t->root, pos, p, T, Rp, row);
}

static int cmp_i32(const void *a, const void *b)
{
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* counts[k] = |N(queries[k])| (queries == NULL: queries[k] = k). */
void orc_count(const orc_tree *t, const double *pos, const double *h,
               const int64_t *queries, int64_t nq, int32_t *counts, int nthreads)
{
    (void)nthreads;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t k = 0; k < nq; k++) {
        orc_row row = {NULL, 0, 0};
        one_row(t, pos, h, queries ? queries[k] : k, &row);
        counts[k] = (int32_t)row.len;
    }
}

/* Rows of the listed queries, each sorted ascending, written at            */
/* idx[offsets[k] .. offsets[k+1]) (offsets from a previous orc_count).     */
/* Returns 0, or -1 if a row does not fit its slot.                         */
int orc_rows(const orc_tree *t, const double *pos, const double *h,
             const int64_t *queries, int64_t nq, const int64_t *offsets,
             int32_t *idx, int nthreads)
{
    int bad = 0;
    (void)nthreads;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads > 0 ? nthreads : 1) reduction(| : bad)
    for (int64_t k = 0; k < nq; k++) {
        orc_row row = {idx + offsets[k], offsets[k + 1] - offsets[k], 0};
        one_row(t, pos, h, queries ? queries[k] : k, &row);
        if (row.len != row.cap)
            bad |= 1;
        else
            qsort(row.buf, (size_t)row.len, sizeof(int32_t), cmp_i32);
    }
    return bad ? -1 : 0;
}

/* ------------------------------------------------------------------ */
/* O(n^2) brute force: the plain definition of the result. */
/* Written separately from the tree path: every j in [0,n), j != i.     */
/* ------------------------------------------------------------------ */
void orc_brute_count(const double *pos, const double *h, int64_t n,
                     const int64_t *queries, int64_t nq, int32_t *counts, int nthreads)
{
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t k = 0; k < nq; k++) {
        int64_t i = queries ? queries[k] : k;
        double two_h = 2.0 * h[i];
        double T = two_h * two_h;
        int32_t c = 0;
        for (int64_t j = 0; j < n; j++) {
            if (j == i)
                continue;
            double dx = pos[3 * i + 0] - pos[3 * j + 0];
            double dy = pos[3 * i + 1] - pos[3 * j + 1];
            double dz = pos[3 * i + 2] - pos[3 * j + 2];
            if ((dx * dx + dy * dy) + dz * dz < T)
                c++;
        }
        counts[k] = c;
    }
}

/* Rows ascending by construction (j increases). */
int orc_brute_rows(const double *pos, const double *h, int64_t n,
                   const int64_t *queries, int64_t nq, const int64_t *offsets,
                   int32_t *idx, int nthreads)
{
    int bad = 0;
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1) reduction(| : bad)
    for (int64_t k = 0; k < nq; k++) {
        int64_t i = queries ? queries[k] : k;
        double two_h = 2.0 * h[i];
        double T = two_h * two_h;
        int64_t w = offsets[k], end = offsets[k + 1];
        for (int64_t j = 0; j < n; j++) {
            if (j == i)
                continue;
            double dx = pos[3 * i + 0] - pos[3 * j + 0];
            double dy = pos[3 * i + 1] - pos[3 * j + 1];
            double dz = pos[3 * i + 2] - pos[3 * j + 2];
            if ((dx * dx + dy * dy) + dz * dz < T) {
                if (w < end) idx[w] = (int32_t)j;
                w++;
            }
        }
        if (w != end)
            bad |= 1;
    }
    return bad ? -1 : 0;
}

/* ------------------------------------------------------------------ */
/* Symmetric criterion (reading R22, not in the      */
/* paper, whose Alg. 2 uses the query's h_p only  */
/* leaves it open): j != i is a neighbor of i iff                       */
/*   ((dx*dx + dy*dy) + dz*dz) < t*t,  t = 2 max(h_i, h_j)             */
/* in fp64 (max is exact).  The plain definition, O(n^2), every j.      */
/* ------------------------------------------------------------------ */
static int orc_sym_pair(const double *pos, const double *h, int64_t i, int64_t j)
{
    double hm = h[i] > h[j] ? h[i] : h[j];
    double t = 2.0 * hm;
    double dx = pos[3 * i + 0] - pos[3 * j + 0];
    double dy = pos[3 * i + 1] - pos[3 * j + 1];
    double dz = pos[3 * i + 2] - pos[3 * j + 2];
    return (dx * dx + dy * dy) + dz * dz < t * t;
}

void orc_brute_count_sym(const double *pos, const double *h, int64_t n,
                         const int64_t *queries, int64_t nq, int32_t *counts, int nthreads)
{
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t k = 0; k < nq; k++) {
        int64_t i = queries ? queries[k] : k;
        int32_t c = 0;
        for (int64_t j = 0; j < n; j++)
            if (j != i && orc_sym_pair(pos, h, i, j))
                c++;
        counts[k] = c;
    }
}

int orc_brute_rows_sym(const double *pos, const double *h, int64_t n,
                       const int64_t *queries, int64_t nq, const int64_t *offsets,
                       int32_t *idx, int nthreads)
{
    int bad = 0;
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1) reduction(| : bad)
    for (int64_t k = 0; k < nq; k++) {
        int64_t i = queries ? queries[k] : k;
        int64_t w = offsets[k], end = offsets[k + 1];
        for (int64_t j = 0; j < n; j++) {
            if (j != i && orc_sym_pair(pos, h, i, j)) {
                if (w < end) idx[w] = (int32_t)j;
                w++;
            }
        }
        if (w != end)
            bad |= 1;
    }
    return bad ? -1 : 0;
}

/* ------------------------------------------------------------------ */
/* SPH density consumer (the paper's use of the     */
/* neighbor lists, Sec. I P:50-56 and Sec. IV-H).  Reading    */
/* R21 (not in the paper): the M4 cubic spline of compact support 2h,   */
/*   W(r, h) = w(r / h) / (pi h^3),                                     */
/*   w(q) = 1 - 1.5 q^2 + 0.75 q^3 (0 <= q < 1),  0.25 (2 - q)^3        */
/*   (1 <= q < 2),  0 (q >= 2),                                         */
/* and rho_i = m_i W(0, h_i) + sum_{j in N(i)} m_j W(r_ij, h_i), the     */
/* gather form with the query's h (R13), r_ij = sqrt of the predicate's */
/* d^2 = ((dx*dx + dy*dy) + dz*dz).  Plain fp64.                         */
/* ------------------------------------------------------------------ */
#define ORC_PI 3.14159265358979323846

double orc_w_m4(double q)
{
    if (q < 1.0)
        return 1.0 - 1.5 * q * q + 0.75 * q * q * q;
    if (q < 2.0) {
        double t = 2.0 - q;
        return 0.25 * t * t * t;
    }
    return 0.0;
}

static double pair_r(const double *xi, const double *xj)
{
    double dx = xi[0] - xj[0];
    double dy = xi[1] - xj[1];
    double dz = xi[2] - xj[2];
    return sqrt((dx * dx + dy * dy) + dz * dz);
}

/* rho of the listed queries through the tree walk (rows ascending). */
void orc_density(const orc_tree *t, const double *pos, const double *h, const double *mass,
                 const int64_t *queries, int64_t nq, double *rho, int nthreads)
{
    (void)nthreads;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t k = 0; k < nq; k++) {
        int64_t i = queries ? queries[k] : k;
        orc_row row = {NULL, 0, 0};
        one_row(t, pos, h, i, &row); /* count */
        int32_t *buf = (int32_t *)malloc(sizeof(int32_t) * (size_t)(row.len > 0 ? row.len : 1));
        orc_row full = {buf, row.len, 0};
        one_row(t, pos, h, i, &full);
        qsort(buf, (size_t)full.len, sizeof(int32_t), cmp_i32);
        double sum = mass[i] * orc_w_m4(0.0);
        for (int64_t a = 0; a < full.len; a++) {
            int64_t j = buf[a];
            sum += mass[j] * orc_w_m4(pair_r(pos + 3 * i, pos + 3 * j) / h[i]);
        }
        free(buf);
        rho[k] = sum / (ORC_PI * h[i] * h[i] * h[i]);
    }
}

/* The same sum by the plain definition: every j != i passing the predicate. */
void orc_brute_density(const double *pos, const double *h, const double *mass, int64_t n,
                       const int64_t *queries, int64_t nq, double *rho, int nthreads)
{
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t k = 0; k < nq; k++) {
        int64_t i = queries ? queries[k] : k;
        double two_h = 2.0 * h[i];
        double T = two_h * two_h;
        double sum = mass[i] * orc_w_m4(0.0);
        for (int64_t j = 0; j < n; j++) {
            if (j == i)
                continue;
            double dx = pos[3 * i + 0] - pos[3 * j + 0];
            double dy = pos[3 * i + 1] - pos[3 * j + 1];
            double dz = pos[3 * i + 2] - pos[3 * j + 2];
            double d2 = (dx * dx + dy * dy) + dz * dz;
            if (d2 < T)
                sum += mass[j] * orc_w_m4(sqrt(d2) / h[i]);
        }
        rho[k] = sum / (ORC_PI * h[i] * h[i] * h[i]);
    }
}

int orc_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
