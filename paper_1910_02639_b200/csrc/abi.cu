// abi.cu -- the extern "C" boundary declared in include/btree.h: argument
// validation, error codes, the per-thread stream, stream-ordered allocation,
// phase profiling with CUDA events, and the host-buffer end-to-end call.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <unordered_map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

struct bt_tree {
    bt::TreeDev t;
};

namespace bt {

namespace {
thread_local cudaStream_t g_stream = cudaStreamPerThread;
thread_local std::string g_err;
thread_local int g_status = BT_OK;

std::mutex g_prof_mu;
bool g_prof_on = false;
struct ProfEntry {
    double ms = 0.0;
    int64_t launches = 0;
};
std::map<std::string, ProfEntry> g_prof;
struct Pending {
    std::string name;
    cudaEvent_t a, b;
};
thread_local std::vector<Pending> g_pending;
thread_local std::vector<cudaEvent_t> g_event_pool;

cudaEvent_t get_event() {
    if (!g_event_pool.empty()) {
        cudaEvent_t e = g_event_pool.back();
        g_event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    BT_CUDA(cudaEventCreate(&e));
    return e;
}

void resolve_pending() {
    for (auto &p : g_pending) {
        float ms = 0.f;
        if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
            std::lock_guard<std::mutex> lk(g_prof_mu);
            g_prof[p.name].ms += ms;
        }
        g_event_pool.push_back(p.a);
        g_event_pool.push_back(p.b);
    }
    g_pending.clear();
}

void set_error(int code, const std::string &msg) {
    g_status = code;
    g_err = msg;
}

template <class F>
int guarded(F &&f) {
    try {
        f();
        resolve_pending();
        g_status = BT_OK;
        return BT_OK;
    } catch (const Error &e) {
        g_pending.clear();
        set_error(e.code, e.what());
        return e.code;
    } catch (const std::bad_alloc &) {
        set_error(BT_ERR_OOM, "host allocation failed");
        return BT_ERR_OOM;
    } catch (const std::exception &e) {
        set_error(BT_ERR_CUDA, e.what());
        return BT_ERR_CUDA;
    }
}
}  // namespace

cudaStream_t stream() { return g_stream; }

void after_launch(const char *name) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(BT_ERR_CUDA, std::string("launch of ") + name + ": " + cudaGetErrorString(e));
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof[std::string("kernel.") + name].launches++;
}

Phase::Phase(const char *n) : name(n), on(g_prof_on) {
    if (!on) return;
    a = get_event();
    b = get_event();
    BT_CUDA(cudaEventRecord(a, g_stream));
}
Phase::~Phase() {
    if (!on) return;
    if (cudaEventRecord(b, g_stream) == cudaSuccess) g_pending.push_back(Pending{name, a, b});
}

// Device memory: a per-thread caching allocator over cudaMalloc.  Freed blocks
// are kept and handed out again (best fit, at most 2x the request) to later
// calls of the same thread on the same device, whose work is ordered on the
// same stream -- the stream-ordered pool (cudaMallocAsync) re-mapped physical
// memory on every build here (~5 ms per GB), which dominated small steps.
// Blocks are keyed by the device current at allocation (cudaGetDevice), so a
// thread that switches devices never receives another GPU's memory.  On OOM
// the cache is released and the allocation retried once.
namespace {
int current_device() {
    int d = 0;
    BT_CUDA(cudaGetDevice(&d));
    return d;
}
struct BlockCache {
    std::map<int, std::multimap<size_t, void *>> free_blocks;    // per device
    std::unordered_map<void *, std::pair<int, size_t>> owner;    // block -> (device, size)
    void release_all() {
        cudaStreamSynchronize(g_stream);
        int cur = 0;
        cudaGetDevice(&cur);
        for (auto &dv : free_blocks) {
            cudaSetDevice(dv.first);
            for (auto &kv : dv.second) {
                cudaFree(kv.second);
                owner.erase(kv.second);
            }
            dv.second.clear();
        }
        cudaSetDevice(cur);
    }
    ~BlockCache() {
        for (auto &dv : free_blocks) {
            cudaSetDevice(dv.first);
            for (auto &kv : dv.second) cudaFree(kv.second);
        }
    }
};
BlockCache &block_cache() {
    thread_local BlockCache c;
    return c;
}
size_t round_block(size_t bytes) {
    if (bytes < 512) return 512;
    if (bytes < (1u << 20)) return (bytes + 511) & ~size_t(511);
    return (bytes + (2u << 20) - 1) & ~size_t((2u << 20) - 1);
}
}  // namespace

void *dmalloc(size_t bytes) {
    BlockCache &C = block_cache();
    const int dev = current_device();
    const size_t want = round_block(bytes);
    auto &fb = C.free_blocks[dev];
    auto it = fb.lower_bound(want);
    if (it != fb.end() && it->first <= 2 * want) {
        void *p = it->second;
        fb.erase(it);
        return p;
    }
    static const bool trace = getenv("BT_TRACE") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        C.release_all();
        e = cudaMalloc(&p, want);
    }
    if (trace) {
        double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        fprintf(stderr, "[bt] cudaMalloc %zu bytes on device %d: %.1f us\n", want, dev, us);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw Error(e == cudaErrorMemoryAllocation ? BT_ERR_OOM : BT_ERR_CUDA,
                    "device allocation of " + std::to_string(bytes) + " bytes: " + cudaGetErrorString(e));
    }
    C.owner[p] = {dev, want};
    return p;
}
void dfree(void *p) {
    if (!p) return;
    BlockCache &C = block_cache();
    auto it = C.owner.find(p);
    if (it == C.owner.end()) {  // allocated by another thread: return it to the driver
        cudaStreamSynchronize(g_stream);
        cudaFree(p);
        return;
    }
    C.free_blocks[it->second.first].emplace(it->second.second, p);
}

int num_sms() {
    static int v[128] = {0};
    const int dev = current_device();
    if (dev < 0 || dev >= 128) throw Error(BT_ERR_CUDA, "device ordinal out of range");
    if (!v[dev]) BT_CUDA(cudaDeviceGetAttribute(&v[dev], cudaDevAttrMultiProcessorCount, dev));
    return v[dev];
}

int release_cache() {
    block_cache().release_all();
    return 0;
}

HostScratch &host_scratch() {
    thread_local HostScratch hs;
    return hs;
}

void read_back(std::initializer_list<ReadBack> items) {
    char *buf = reinterpret_cast<char *>(host_scratch().p);
    size_t off = 0;
    for (const auto &it : items) {
        if (off + it.bytes > 64 * sizeof(int64_t)) throw Error(BT_ERR_CUDA, "read_back: scratch too small");
        BT_CUDA(cudaMemcpyAsync(buf + off, it.src, it.bytes, cudaMemcpyDeviceToHost, g_stream));
        off += (it.bytes + 15) & ~size_t(15);
    }
    BT_CUDA(cudaStreamSynchronize(g_stream));
    off = 0;
    for (const auto &it : items) {
        memcpy(it.dst, buf + off, it.bytes);
        off += (it.bytes + 15) & ~size_t(15);
    }
}

}  // namespace bt

using namespace bt;

extern "C" {

bt_tree *bt_build_policy(const double *pos, int64_t n, int32_t bucket_size, double max_empty, double alpha,
                         int32_t depth_cap, int32_t policy) {
    if (policy < BT_POLICY_BTREE || policy > BT_POLICY_QUADTREE) {
        set_error(BT_ERR_ARG, "bt_build_policy: policy must be BT_POLICY_BTREE, _OCTREE, _BTREE_2D or _QUADTREE");
        return nullptr;
    }
    if (n < 0 || n > 2147483647LL || (pos == nullptr && n > 0) || bucket_size < 1 || !(max_empty > 0.0 && max_empty <= 1.0) ||
        !(alpha >= 0.0 && alpha <= 1.0) || depth_cap < 0 || depth_cap > 1000) {
        set_error(BT_ERR_ARG,
                  "bt_build: need 0 <= n <= 2^31-1, pos != NULL, bucket_size >= 1, max_empty in (0,1], alpha in [0,1], "
                  "0 <= depth_cap <= 1000");
        return nullptr;
    }
    bt_tree *t = nullptr;
    int rc = guarded([&] {
        t = new bt_tree();
        t->t.n = n;
        t->t.s = bucket_size;
        t->t.beta = max_empty;
        t->t.alpha = alpha;
        t->t.depth_cap = depth_cap;
        t->t.octree = policy == BT_POLICY_OCTREE || policy == BT_POLICY_QUADTREE;
        t->t.dims = (policy == BT_POLICY_BTREE_2D || policy == BT_POLICY_QUADTREE) ? 2 : 3;
        Phase ph("build.total");
        build_tree(t->t, pos);
        BT_CUDA(cudaStreamSynchronize(stream()));
    });
    if (rc != BT_OK) {
        if (t) {
            std::string msg = g_err;
            delete t;
            cudaStreamSynchronize(stream());
            g_err = msg;
            g_status = rc;
        }
        return nullptr;
    }
    return t;
}

bt_tree *bt_build_ex(const double *pos, int64_t n, int32_t bucket_size, double max_empty, double alpha,
                     int32_t depth_cap) {
    return bt_build_policy(pos, n, bucket_size, max_empty, alpha, depth_cap, BT_POLICY_BTREE);
}

bt_tree *bt_build(const double *pos, int64_t n, int32_t bucket_size, double max_empty) {
    return bt_build_ex(pos, n, bucket_size, max_empty, 0.5, 64);
}

int bt_find_neighbors(const bt_tree *tc, const double *h, int32_t ngmax, int32_t *counts, int64_t *offsets,
                      int32_t *nbr_idx) {
    bt_tree *t = const_cast<bt_tree *>(tc);
    if (!t || ngmax < 1 || (t->t.n > 0 && (!h || !counts || !offsets)) || (t->t.n == 0 && !offsets)) {
        set_error(BT_ERR_ARG, "bt_find_neighbors: need a tree, h, counts, offsets and ngmax >= 1");
        return BT_ERR_ARG;
    }
    return guarded([&] {
        Phase ph("search.total");
        const int64_t cap = t->t.n * (int64_t)ngmax;
        t->t.ngmax = ngmax;
        find_neighbors(t->t, h, counts, offsets, nbr_idx, cap, true, nbr_idx != nullptr);
    });
}

int bt_fill_neighbors(const bt_tree *tc, const double *h, const int64_t *offsets, int32_t *nbr_idx, int64_t capacity) {
    bt_tree *t = const_cast<bt_tree *>(tc);
    if (!t || (t->t.n > 0 && (!h || !offsets || (!nbr_idx && capacity > 0))) || capacity < 0) {
        set_error(BT_ERR_ARG, "bt_fill_neighbors: need a tree, h, offsets, nbr_idx and capacity >= 0");
        return BT_ERR_ARG;
    }
    return guarded([&] {
        Phase ph("search.total");
        if (t->t.n == 0) return;
        find_neighbors(t->t, h, nullptr, const_cast<int64_t *>(offsets), nbr_idx, capacity, false, true);
    });
}

int bt_find_neighbors_sym(const bt_tree *tc, const double *h, int32_t ngmax, int32_t *counts, int64_t *offsets,
                          int32_t *nbr_idx) {
    bt_tree *t = const_cast<bt_tree *>(tc);
    if (!t || ngmax < 1 || (t->t.n > 0 && (!h || !counts || !offsets)) || (t->t.n == 0 && !offsets)) {
        set_error(BT_ERR_ARG, "bt_find_neighbors_sym: need a tree, h, counts, offsets and ngmax >= 1");
        return BT_ERR_ARG;
    }
    return guarded([&] {
        Phase ph("search.total");
        const int64_t cap = t->t.n * (int64_t)ngmax;
        t->t.ngmax = ngmax;
        find_neighbors(t->t, h, counts, offsets, nbr_idx, cap, true, nbr_idx != nullptr, true);
    });
}

int bt_fill_neighbors_sym(const bt_tree *tc, const double *h, const int64_t *offsets, int32_t *nbr_idx,
                          int64_t capacity) {
    bt_tree *t = const_cast<bt_tree *>(tc);
    if (!t || (t->t.n > 0 && (!h || !offsets || (!nbr_idx && capacity > 0))) || capacity < 0) {
        set_error(BT_ERR_ARG, "bt_fill_neighbors_sym: need a tree, h, offsets, nbr_idx and capacity >= 0");
        return BT_ERR_ARG;
    }
    return guarded([&] {
        Phase ph("search.total");
        if (t->t.n == 0) return;
        find_neighbors(t->t, h, nullptr, const_cast<int64_t *>(offsets), nbr_idx, capacity, false, true, true);
    });
}

int bt_set_partition(bt_tree *t, int32_t part, int32_t nparts) {
    if (!t || nparts < 1 || part < 0 || part >= nparts) {
        set_error(BT_ERR_ARG, "bt_set_partition: need a tree, nparts >= 1 and 0 <= part < nparts");
        return BT_ERR_ARG;
    }
    t->t.part = part;
    t->t.nparts = nparts;
    t->t.rec_valid = false;  // the recorded masks belong to the previous unit range
    return BT_OK;
}

int bt_set_tree_order(bt_tree *t, int on) {
    if (!t) {
        set_error(BT_ERR_ARG, "bt_set_tree_order: NULL tree");
        return BT_ERR_ARG;
    }
    t->t.tree_order = on != 0;
    t->t.rec_valid = false;  // the recorded candidates hold the other space's indices
    return BT_OK;
}

namespace bt_export {
__global__ void reorder_kernel(const double4 *rec, const double *src, int ncomp, int64_t n, double *dst) {
    const int64_t total = n * ncomp;
    if (ncomp == 1) {
        for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
            dst[k] = src[__double_as_longlong(rec[k].w)];
        return;
    }
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = e / ncomp, c = e - k * ncomp;
        dst[e] = src[__double_as_longlong(rec[k].w) * ncomp + c];
    }
}
}  // namespace bt_export

int bt_reorder(const bt_tree *t, const double *src, int32_t ncomp, double *dst) {
    if (!t || ncomp < 1 || ncomp > 16 || (t->t.n > 0 && (!src || !dst))) {
        set_error(BT_ERR_ARG, "bt_reorder: need a tree, src, dst and 1 <= ncomp <= 16");
        return BT_ERR_ARG;
    }
    return guarded([&] {
        const TreeDev &d = t->t;
        cudaStream_t st = stream();
        if (d.n) {
            bt_export::reorder_kernel<<<grid_for(d.n * ncomp, 256, (int64_t)num_sms() * 16), 256, 0, st>>>(
                d.rec.p, src, ncomp, d.n, dst);
            BT_LAUNCH("reorder");
        }
        BT_CUDA(cudaStreamSynchronize(st));
    });
}

int bt_density(const bt_tree *tc, const double *h, const double *mass, double *rho) {
    bt_tree *t = const_cast<bt_tree *>(tc);
    if (!t || (t->t.n > 0 && (!h || !mass || !rho))) {
        set_error(BT_ERR_ARG, "bt_density: need a tree, h, mass and rho");
        return BT_ERR_ARG;
    }
    return guarded([&] {
        Phase ph("density.total");
        density(t->t, h, mass, rho);
        BT_CUDA(cudaStreamSynchronize(stream()));
    });
}

void bt_free(bt_tree *t) {
    if (!t) return;
    delete t;  // DBuf destructors return the blocks to this thread's cache
    cudaStreamSynchronize(stream());
}

int bt_search_host(const double *pos_h, const double *h_h, int64_t n, int32_t bucket_size, double max_empty,
                   int32_t *counts_h, int64_t *offsets_h, int32_t *nbr_h, int64_t capacity) {
    if (n < 0 || (n > 0 && (!pos_h || !h_h || !counts_h)) || !offsets_h || capacity < 0 || (capacity > 0 && !nbr_h)) {
        set_error(BT_ERR_ARG, "bt_search_host: invalid arguments");
        return BT_ERR_ARG;
    }
    bt_tree *t = nullptr;
    int rc = guarded([&] {
        cudaStream_t st = stream();
        // a side stream carries the copies that do not gate the next kernel:
        // h's upload overlaps the build, counts / offsets go home during the fill
        static thread_local std::map<int, cudaStream_t> sides;  // one per device
        cudaStream_t &side = sides[current_device()];
        if (!side) BT_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
        cudaEvent_t ev_h, ev_c;
        BT_CUDA(cudaEventCreateWithFlags(&ev_h, cudaEventDisableTiming));
        BT_CUDA(cudaEventCreateWithFlags(&ev_c, cudaEventDisableTiming));
        struct Events {
            cudaEvent_t a, b;
            ~Events() { cudaEventDestroy(a); cudaEventDestroy(b); }
        } evs{ev_h, ev_c};
        Phase ph("e2e.total");
        DBuf<double> pos(3 * (size_t)n), h((size_t)n);
        DBuf<int32_t> counts((size_t)n);
        DBuf<int64_t> offsets((size_t)n + 1);
        struct SideSync {  // (declared after the buffers: on any exit the side stream drains first)
            cudaStream_t s;
            ~SideSync() { cudaStreamSynchronize(s); }
        } side_sync{side};
        BT_CUDA(cudaEventRecord(ev_h, st));  // the buffers exist before the side stream writes them
        BT_CUDA(cudaStreamWaitEvent(side, ev_h, 0));
        if (n) BT_CUDA(cudaMemcpyAsync(pos.p, pos_h, 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
        if (n) BT_CUDA(cudaMemcpyAsync(h.p, h_h, n * sizeof(double), cudaMemcpyHostToDevice, side));
        BT_CUDA(cudaEventRecord(ev_h, side));
        t = bt_build(pos.p, n, bucket_size, max_empty);
        if (!t) throw Error(g_status, g_err);
        BT_CUDA(cudaStreamWaitEvent(st, ev_h, 0));  // h has arrived
        find_neighbors(t->t, h.p, counts.p, offsets.p, nullptr, 0, true, false);
        const int64_t total = t->t.total_pairs;
        BT_CUDA(cudaEventRecord(ev_c, st));
        BT_CUDA(cudaStreamWaitEvent(side, ev_c, 0));
        if (n) BT_CUDA(cudaMemcpyAsync(counts_h, counts.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, side));
        BT_CUDA(cudaMemcpyAsync(offsets_h, offsets.p, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, side));
        BT_CUDA(cudaEventRecord(ev_c, side));
        if (total > capacity) {
            BT_CUDA(cudaStreamSynchronize(side));
            BT_CUDA(cudaStreamSynchronize(st));
            throw Error(BT_ERR_CAPACITY, "bt_search_host: " + std::to_string(total) + " pairs exceed capacity " +
                                             std::to_string(capacity));
        }
        DBuf<int32_t> nbr((size_t)(total > 0 ? total : 1));
        find_neighbors(t->t, h.p, nullptr, offsets.p, nbr.p, total, false, true);
        if (total) BT_CUDA(cudaMemcpyAsync(nbr_h, nbr.p, total * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        BT_CUDA(cudaStreamWaitEvent(st, ev_c, 0));  // (buffers are released on st)
        BT_CUDA(cudaStreamSynchronize(st));
    });
    if (t) {
        std::string msg = g_err;
        int s = g_status;
        bt_free(t);
        g_err = msg;
        g_status = s;
    }
    return rc;
}

int bt_set_stream(void *s) {
    g_stream = s ? (cudaStream_t)s : cudaStreamPerThread;
    g_status = BT_OK;
    return BT_OK;
}

int bt_release_cache(void) {
    return guarded([&] { release_cache(); });
}

int bt_set_exact_only(int on) {
    set_exact_only(on != 0);
    g_status = BT_OK;
    return BT_OK;
}

const char *bt_last_error(void) { return g_err.c_str(); }
int bt_last_status(void) { return g_status; }

int bt_tree_stats(const bt_tree *t, bt_stats *out) {
    if (!t || !out) {
        set_error(BT_ERR_ARG, "bt_tree_stats: NULL argument");
        return BT_ERR_ARG;
    }
    const TreeDev &d = t->t;
    std::memset(out, 0, sizeof(*out));
    out->n = d.n;
    out->nodes = d.n_nodes;
    out->leaves = d.n_leaves;
    out->halvings = d.halvings;
    out->overfull = d.overfull;
    out->max_leaf = d.max_leaf;
    out->depth = d.depth;
    out->root_b = d.root_b;
    out->units = d.n_units;
    for (int l = 0; l < 3; l++) {
        out->box_lo[l] = d.box_lo[l];
        out->box_hi[l] = d.box_hi[l];
    }
    out->total_pairs = d.total_pairs;
    out->max_count = d.max_count;
    out->staged = d.staged;
    out->tests = d.tests;
    out->exact_tests = d.exact_tests;
    out->loaded = d.loaded;
    out->mask_words = d.mask_words;
    out->cand_slots = d.cand_slots;
    out->list_entries = d.list_entries;
    out->big_units = d.big_units;
    out->rows_over_ngmax = d.rows_over_ngmax;
    out->mask_words_nonzero = d.mask_words_nz;
    return BT_OK;
}

namespace bt_export {
__global__ void export_perm_kernel(const double4 *rec, int64_t n, int32_t *perm) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        perm[k] = (int32_t)__double_as_longlong(rec[k].w);
}
__global__ void widen_kernel(const int32_t *a, int64_t *b, int64_t n) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        b[k] = a[k];
}
}  // namespace bt_export
using namespace bt_export;

int bt_tree_order(const bt_tree *t, int32_t *perm, int64_t *leaf_begin, int32_t *leaf_count, int32_t *leaf_depth) {
    if (!t) {
        set_error(BT_ERR_ARG, "bt_tree_order: NULL tree");
        return BT_ERR_ARG;
    }
    return guarded([&] {
        const TreeDev &d = t->t;
        cudaStream_t st = stream();
        if (perm && d.n) {
            export_perm_kernel<<<grid_for(d.n, 256, 4096), 256, 0, st>>>(d.rec.p, d.n, perm);
            BT_LAUNCH("export_perm");
        }
        if (leaf_begin && d.n_leaves) {
            widen_kernel<<<grid_for(d.n_leaves, 256, 4096), 256, 0, st>>>(d.leaf_begin.p, leaf_begin, d.n_leaves);
            BT_LAUNCH("export_leaf_begin");
        }
        if (leaf_count && d.n_leaves)
            BT_CUDA(cudaMemcpyAsync(leaf_count, d.leaf_count.p, d.n_leaves * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        if (leaf_depth && d.n_leaves)
            BT_CUDA(cudaMemcpyAsync(leaf_depth, d.leaf_depth.p, d.n_leaves * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        BT_CUDA(cudaStreamSynchronize(st));
    });
}

int bt_profile_enable(int on) {
    g_prof_on = on != 0;
    return BT_OK;
}

int bt_profile_reset(void) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.clear();
    return BT_OK;
}

int bt_profile_get(int max_entries, const char **names, double *ms, int64_t *launches) {
    static thread_local std::vector<std::string> keep;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    keep.clear();
    int k = 0;
    for (auto &kv : g_prof) {
        if (k < max_entries) {
            keep.push_back(kv.first);
        }
        k++;
    }
    int i = 0;
    for (auto &kv : g_prof) {
        if (i >= max_entries) break;
        if (names) names[i] = keep[i].c_str();
        if (ms) ms[i] = kv.second.ms;
        if (launches) launches[i] = kv.second.launches;
        i++;
    }
    return k;
}

}  // extern "C"
