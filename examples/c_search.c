/*
 * c_search.c -- the C ABI used from plain C (no Python, no PyTorch):
 * host buffers in, exact neighbor lists out, through bt_search_host; then the
 * device-pointer path (cudaMalloc'd pos/h) through bt_build /
 * bt_find_neighbors / bt_fill_neighbors / bt_tree_stats / bt_free.
 * Checks a few rows against a direct double loop with the same predicate.
 *
 *   gcc -O2 -std=c11 -ffp-contract=off examples/c_search.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_1910_02639_b200 -lbtree -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1910_02639_b200 -o c_search && ./c_search [n]
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "btree.h"

static double urand(uint64_t *s) { /* splitmix64 -> [0, 1) */
    uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return (double)((z ^ (z >> 31)) >> 11) * 0x1p-53;
}

static int64_t brute_count(const double *pos, const double *h, int64_t n, int64_t i) {
    double t = 2.0 * h[i], T = t * t;
    int64_t c = 0;
    for (int64_t j = 0; j < n; j++) {
        if (j == i) continue;
        double dx = pos[3 * i] - pos[3 * j], dy = pos[3 * i + 1] - pos[3 * j + 1], dz = pos[3 * i + 2] - pos[3 * j + 2];
        if ((dx * dx + dy * dy) + dz * dz < T) c++; /* compiled with -ffp-contract=off */
    }
    return c;
}

int main(int argc, char **argv) {
    int64_t n = argc > 1 ? atoll(argv[1]) : 100000;
    double *pos = malloc(sizeof(double) * 3 * n), *h = malloc(sizeof(double) * n);
    uint64_t s = 1234;
    for (int64_t i = 0; i < 3 * n; i++) pos[i] = urand(&s);
    for (int64_t i = 0; i < n; i++) h[i] = 0.015 * (0.8 + 0.4 * urand(&s)); /* ~11 neighbours at n = 1e5 */
    int32_t *counts = malloc(sizeof(int32_t) * n);
    int64_t *offsets = malloc(sizeof(int64_t) * (n + 1));
    int64_t cap = n * 64;
    int32_t *nbr = malloc(sizeof(int32_t) * cap);
    /* 1. host buffers, one call */
    int rc = bt_search_host(pos, h, n, 64, 0.5, counts, offsets, nbr, cap);
    if (rc != BT_OK) { fprintf(stderr, "bt_search_host: %s\n", bt_last_error()); return 1; }
    for (int64_t i = 0; i < n; i += n / 7 + 1)
        if (counts[i] != brute_count(pos, h, n, i)) { fprintf(stderr, "count mismatch at %lld\n", (long long)i); return 1; }
    /* 2. device pointers */
    double *dpos, *dh;
    int32_t *dcounts, *dnbr;
    int64_t *doff;
    cudaMalloc((void **)&dpos, sizeof(double) * 3 * n);
    cudaMalloc((void **)&dh, sizeof(double) * n);
    cudaMalloc((void **)&dcounts, sizeof(int32_t) * n);
    cudaMalloc((void **)&doff, sizeof(int64_t) * (n + 1));
    cudaMemcpy(dpos, pos, sizeof(double) * 3 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dh, h, sizeof(double) * n, cudaMemcpyHostToDevice);
    bt_tree *t = bt_build(dpos, n, 64, 0.5);
    if (!t) { fprintf(stderr, "bt_build: %s\n", bt_last_error()); return 1; }
    if (bt_find_neighbors(t, dh, 1, dcounts, doff, NULL) != BT_OK) { fprintf(stderr, "%s\n", bt_last_error()); return 1; }
    int64_t total;
    cudaMemcpy(&total, doff + n, sizeof(int64_t), cudaMemcpyDeviceToHost);
    cudaMalloc((void **)&dnbr, sizeof(int32_t) * (total > 0 ? total : 1));
    if (bt_fill_neighbors(t, dh, doff, dnbr, total) != BT_OK) { fprintf(stderr, "%s\n", bt_last_error()); return 1; }
    bt_stats st;
    bt_tree_stats(t, &st);
    printf("n=%lld pairs=%lld (host call: %lld) depth=%d root_b=%d leaves=%lld max_count=%lld\n", (long long)n,
           (long long)total, (long long)offsets[n], st.depth, st.root_b, (long long)st.leaves, (long long)st.max_count);
    bt_free(t);
    cudaFree(dpos); cudaFree(dh); cudaFree(dcounts); cudaFree(doff); cudaFree(dnbr);
    if (total != offsets[n]) { fprintf(stderr, "totals differ\n"); return 1; }
    printf("c_search ok\n");
    return 0;
}
