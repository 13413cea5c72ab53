/* c_api_demo.c — MegaScan's analysis through the C ABI only (include/megascan/scan.h), no Python.
 *
 * Builds a 2-rank job (TP=1, PP=1, DP=2) in host memory: every iteration both ranks run one compute
 * kernel and join one all-reduce; rank 1's kernel is 3x slower. Then: load, analyze, export the
 * per-event waits and the per-rank verdicts, and print them.
 *   gcc -O2 -I include examples/c_api_demo.c -L paper_2507_19845_b200 -lmegascan \
 *       -Wl,-rpath,$PWD/paper_2507_19845_b200 -o c_api_demo && ./c_api_demo                          */
#include <stdio.h>
#include <stdlib.h>

#include "megascan/scan.h"

#define ITERS 12
#define CHECK(x)                                                                         \
    do {                                                                                 \
        scan_status s_ = (x);                                                            \
        if (s_ < 0) { fprintf(stderr, "%s failed: %d %s\n", #x, s_, scan_last_error(ctx)); return 1; } \
    } while (0)

int main(void) {
    scan_ctx* ctx = NULL;
    if (scan_create(&ctx, 0, NULL) < 0) { fprintf(stderr, "scan_create failed (no CUDA device?)\n"); return 1; }
    enum { PER_RANK = 2 * ITERS, N = 2 * PER_RANK };
    uint64_t rank_off[3] = {0, PER_RANK, N};
    uint32_t dur[N], comm[N], pay[N];
    uint16_t kind[N], meta[N];
    for (int r = 0; r < 2; ++r)
        for (int it = 0; it < ITERS; ++it) {
            const int c = r * PER_RANK + 2 * it, a = c + 1;
            kind[c] = SCAN_KIND_COMPUTE | (7 << 4);                    /* op id 7 */
            dur[c] = r == 1 ? 3000000u : 1000000u;                     /* rank 1: 3 ms instead of 1 ms */
            kind[a] = SCAN_KIND_ALLREDUCE | 8;                          /* iter_end */
            dur[a] = r == 1 ? 200000u : 2200000u;                      /* rank 0 waits 2 ms for rank 1 */
            comm[c] = comm[a] = 0; pay[c] = pay[a] = 0; meta[c] = meta[a] = 0;
        }
    const uint64_t coff[2] = {0, 2};
    const uint32_t cmem[2] = {0, 1};
    const scan_topology topo = {1, 1, 2, 0};
    const scan_comm_table comms = {1, coff, cmem};
    const scan_event_columns cols = {N, rank_off, NULL, dur, kind, meta, comm, pay};
    CHECK(scan_load_events(ctx, &topo, &comms, &cols, SCAN_HOST_PTRS));
    scan_detect_config d = {3, 2, 50000, 3, 10, 10, 0, 0, 0};
    scan_localize_config l = {100000, 7, 10, 7, 10, 10, 3, 0, 0, 100000};
    scan_match_result m;
    scan_detect_result dr;
    scan_localize_result lr;
    CHECK(scan_analyze(ctx, &d, &l, &m, &dr, &lr));
    uint32_t wait[N];
    uint8_t verdict[2], label[2];
    CHECK(scan_export(ctx, SCAN_OUT_EV_WAIT, wait, sizeof wait, 0));
    CHECK(scan_export(ctx, SCAN_OUT_WL_VERDICT, verdict, sizeof verdict, 0));
    CHECK(scan_export(ctx, SCAN_OUT_LB_LABEL, label, sizeof label, 0));
    printf("instances %llu fused %d\n", (unsigned long long)m.n_instances, scan_used_fused(ctx));
    printf("wait rank0 %u rank1 %u\n", wait[1], wait[PER_RANK + 1]);
    printf("verdict %u %u label %u %u\n", verdict[0], verdict[1], label[0], label[1]);
    scan_destroy(ctx);
    /* expected: 12 instances; rank 0 waits 2 ms per all-reduce, rank 1 none; rank 1 ComputeSlow (1), source (1) */
    return (m.n_instances == ITERS && wait[1] == 2000000u && wait[PER_RANK + 1] == 0 && verdict[1] == SCAN_V_COMPUTE_SLOW &&
            label[1] == SCAN_L_SOURCE_RANK) ? 0 : 2;
}
