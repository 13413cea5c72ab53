/*
 * megascan/scan.h — C ABI of the B200-native MegaScan trace-analysis hot path.
 *
 * The operation is MegaScan's analysis pass (§3.2, lines 127-154 of
 * /root/reference/PAPER.md, cited below as P:Lnn): given per-rank CUDA-event
 * operator traces of a TP x PP x DP Megatron job it
 *   (1) matches each collective / P2P instance across the ranks of its
 *       communicator ("Dependency reconstruction"),
 *   (2) derives per-operator compute / wait / transfer times (end-simultaneity,
 *       P:L133; reading R5/R6),
 *   (3) flags slow ranks: stage 1 cross-DP comparison, stage 2
 *       collective start lag, stage 3 P2P effective bandwidth
 *       (P:L150-154),
 *   (4) separates anomaly sources from victims by walking the wait-for
 *       structure (reading R17).
 * Every decision is integer / exact-rational; f64 appears only in reported
 * ratios (reading R19).
 *
 * Conventions
 *  - All functions are extern "C", all integers fixed width.
 *  - Pointers are HOST pointers unless the argument or flag says DEVICE.
 *  - All device work is enqueued on the stream given to scan_create(); every
 *    call returns after its work completed (it synchronises that stream).
 *  - A context is not thread-safe. Result arrays are owned by the context and
 *    stay valid until the next scan_load_events() or scan_destroy().
 *  - Errors: a negative scan_status; scan_last_error() gives a message.
 *    No CPU fallback exists: without a CUDA device every call fails with
 *    SCAN_E_CUDA.
 */
#ifndef MEGASCAN_SCAN_H
#define MEGASCAN_SCAN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t scan_status;
#define SCAN_OK               0
#define SCAN_PARTIAL          1   /* success, but unmatched / inconsistent instances were reported */
#define SCAN_E_INVALID_ARG   -1
#define SCAN_E_SCHEMA        -2   /* event fails the schema (kind, comm id, membership, peer) */
#define SCAN_E_INTEGRITY     -3   /* only with SCAN_STRICT: any unmatched / mismatched instance */
#define SCAN_E_ORDER         -4   /* call sequence violated (detect before match, ...) */
#define SCAN_E_CUDA          -5
#define SCAN_E_NCCL          -6
#define SCAN_E_OOM           -7
#define SCAN_E_UNSUPPORTED   -8   /* a documented capacity limit was exceeded */

typedef struct scan_ctx scan_ctx;

/* ---- event schema (P:L105-114 CUDA-event ops + tracers.scope metadata) ---------------- */
/* kind_op u16 = kind:3 | iter_end:1 | op_id:12                                             */
#define SCAN_KIND_COMPUTE        0
#define SCAN_KIND_ALLREDUCE      1
#define SCAN_KIND_ALLGATHER      2
#define SCAN_KIND_REDUCESCATTER  3
#define SCAN_KIND_BROADCAST      4
#define SCAN_KIND_SEND           5
#define SCAN_KIND_RECV           6
/* meta u16 = mb:10 | chunk:3 | bwd:1 | warmup:1 | rsv:1  (warmup: forward send issued before
   the sender's first backward of its iteration, reading R13)                     */

typedef struct scan_topology {
    int32_t tp, pp, dp;      /* world = tp*pp*dp ranks                                         */
    uint32_t rank_order;     /* must be 0: rank = tp + TP*(dp + DP*pp) (reading R1) */
} scan_topology;

typedef struct scan_comm_table {     /* collective communicators ("global ID list")    */
    uint32_t n_comms;
    const uint64_t* offsets;         /* HOST [n_comms+1], CSR into members                      */
    const uint32_t* members;         /* HOST, ascending rank ids per communicator               */
} scan_comm_table;

typedef struct scan_event_columns {  /* structure-of-arrays, events grouped by rank, program order */
    uint64_t n_events;
    const uint64_t* rank_offsets;    /* HOST [world+1], monotone; rank r owns [off[r], off[r+1]) */
    const int64_t*  start_ns;        /* optional (may be NULL): local-clock start; read only by
                                        scan_align (the analysis never reads it, reading R5)      */
    const uint32_t* dur_ns;          /* CUDA-event duration, ns                                    */
    const uint16_t* kind_op;
    const uint16_t* meta;
    const uint32_t* comm;            /* collective: communicator id; SEND/RECV: peer rank          */
    const uint32_t* payload_bytes;   /* P2P payload; ignored for other kinds                       */
} scan_event_columns;

/* scan_load_events flags */
#define SCAN_HOST_PTRS    0u   /* columns are host memory: copied H2D (pinned memory recommended) */
#define SCAN_DEVICE_PTRS  1u   /* columns are device memory on the ctx device: borrowed, zero-copy;
                                  caller keeps them alive and unchanged until the next load/destroy;
                                  each column must be 16-byte aligned                              */
#define SCAN_STRICT       2u   /* scan_match_collectives returns SCAN_E_INTEGRITY on any report    */

/* ---- results ----------------------------------------------------------------------------- */
typedef struct scan_match_result {
    uint64_t n_events, n_comm_events, n_compute_events;
    uint64_t n_channels, n_p2p_channels, n_instances;
    uint64_t n_incomplete, n_kind_mismatch, n_payload_mismatch;
    uint64_t n_iters;
} scan_match_result;

typedef struct scan_detect_config {   /* stage 1; defaults from SPEC S:L313 as rationals */
    uint32_t slow_num, slow_den;       /* slow iff slow_den*dur > slow_num*ref     (3, 2)            */
    uint64_t slow_margin_ns;           /*      and dur - ref > margin              (50000)           */
    uint32_t cand_num, cand_den;       /* candidate iff cand_den*slow > cand_num*total (3, 10)       */
    uint32_t min_samples;              /*      and total >= min_samples            (10)              */
    uint32_t window_iters;             /* 0 = whole trace, else sliding windows of k iterations      */
    uint32_t want_ref;                 /* 1: also materialise the per-event reference (ref_ns)       */
    uint32_t pad;
} scan_detect_config;

typedef struct scan_detect_result {
    uint64_t n_windows, n_compared, n_slow, n_candidates, n_class_mismatch;
} scan_detect_result;

typedef struct scan_localize_config {  /* stages 2-3 + walk                 */
    uint64_t late_margin_ns;           /* late iff unique last arriver and dmax-dmin > margin (100000) */
    uint32_t late_num, late_den;       /* ComputeSlow iff late_den*late >= late_num*joined (7, 10)    */
    uint32_t bw_num, bw_den;           /* LinkSlow iff bw_den*p_l*t_g < bw_num*p_g*t_l     (7, 10)    */
    uint32_t min_samples;              /* (10)                                                         */
    uint32_t stage2_classes;           /* bit0 TP groups, bit1 DP groups (3)                           */
    uint32_t stage2_mode;              /* 0 CONDITIONAL (reading R11), 1 UNCONDITIONAL   */
    uint32_t pad;
    uint64_t wait_margin_ns;           /* wait-for edge iff wait > margin (100000)                     */
} scan_localize_config;

typedef struct scan_localize_result {
    uint64_t n_windows, n_links, n_link_slow;
    uint64_t n_compute_slow, n_link_slow_ranks, n_both, n_exonerated, n_insufficient;
    uint64_t n_roots, n_victims, n_unattributed, n_edges;
} scan_localize_result;

/* verdicts (per window, rank) */
#define SCAN_V_NONE           0
#define SCAN_V_COMPUTE_SLOW   1
#define SCAN_V_LINK_SLOW      2
#define SCAN_V_BOTH           3
#define SCAN_V_EXONERATED     4
#define SCAN_V_INSUFFICIENT   5
/* labels (per window, rank) */
#define SCAN_L_CLEAN          0
#define SCAN_L_SOURCE_RANK    1
#define SCAN_L_SOURCE_LINK    2
#define SCAN_L_VICTIM         3
#define SCAN_L_UNATTRIBUTED   4
/* instance flags */
#define SCAN_F_COMPLETE     1u
#define SCAN_F_KIND_OK      2u
#define SCAN_F_PAYLOAD_OK   4u
#define SCAN_F_VALID        8u
#define SCAN_F_UNIQUE_LAST 16u
#define SCAN_F_WARMUP      32u

/* ---- lifecycle ------------------------------------------------------------------------- */
/* cuda_stream: a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream), or NULL for the
   legacy default stream. Errors: SCAN_E_INVALID_ARG, SCAN_E_CUDA.                            */
scan_status scan_create(scan_ctx** out, int cuda_device, void* cuda_stream);
void        scan_destroy(scan_ctx* ctx);
const char* scan_last_error(const scan_ctx* ctx);   /* owned by ctx; "" if none               */

/* ---- multi-GPU: iteration-window shards ----------------------------
   One process per GPU. Shard g of n_shards loads, with scan_load_events(), the events of EVERY
   rank for a contiguous block of whole iterations; shards are ordered by iteration (shard g's
   block follows shard g-1's). Iterations are the natural unit: no instance straddles an
   iteration (the tracer records per-iteration step events; reading R30).
   scan_analyze() on a sharded context is a COLLECTIVE call (every shard must call it, same
   configs) that returns the job-wide analysis:
     * per-event outputs (EV_*, COMM_*, SLOW_BITS) cover this shard's events, in its own order;
     * instance ids are the job-wide ids of the unsharded run; this shard's instances are the
       ranges given by CH_SHARD_K0 / CH_SHARD_N; IN_* rows outside them are unspecified;
     * channel, per-rank, per-window, per-link, verdict, walk and edge outputs and all result
       structs are job-wide and identical on every shard (and to the unsharded run).
   Exchange: two small ncclAllGather (per-channel counts, P2P channel bitmap) for the global
   numbering, one grouped ncclSend/ncclRecv all-to-all that ships each P2P instance record
   (12 B) to the shard owning its link (link pid % n_shards), one grouped ncclAllReduce of the
   per-rank / per-window / per-link partial results.
   Preconditions (else SCAN_E_UNSUPPORTED on every shard): the trace is SPMD (fused path), and
   every shard but the last ends on an iteration boundary of every rank with all members of
   every communicator / P2P pair / DP class in step. Besides scan_analyze, scan_align,
   scan_blame (collective calls) and scan_emit_chrome (the shard's own events) run on a sharded
   context; streaming and JSON ingest do not.
   scan_nccl_unique_id: ncclGetUniqueId into out[128]; the caller broadcasts it (e.g. over a
   torch.distributed group) and every shard passes it to scan_create_sharded, which creates
   the context's own NCCL communicator (destroyed by scan_destroy).
   Errors: SCAN_E_INVALID_ARG (n_shards < 1, shard out of range, null id), SCAN_E_NCCL (NCCL
   failure; message in scan_last_error), SCAN_E_CUDA.                                                  */
scan_status scan_nccl_unique_id(uint8_t out[128]);

/* ---- NEXT-1: timeline alignment (readings AL1-AL6) -----
   Maps every rank's local clock onto the reference rank's, using the matched instances as anchors:
   the members of a valid collective instance "logically finish at the same moment".
   AL1 anchors = ends (start_ns + dur_ns) of a rank's collective events (kinds 1-4) of VALID
       instances; P2P excluded.
   AL2 ranks are aligned in BFS levels from the reference over "shares a valid collective instance";
       a rank of level k uses members of levels < k.
   AL3 target = max aligned end over those members; anchor = (local end, target - local end) in
       program order, an end equal to the previous anchor's skipped.
   AL4 offset(t) piecewise linear between anchors (floor of the exact rational), constant outside.
   AL5 aligned start = start + offset(start); ranks not reached keep their clock (level -1).
   Requires: a completed scan_analyze (or scan_match_collectives) and start_ns given at load.
   Outputs SCAN_OUT_AL_*. On a sharded context (scan_create_sharded*) it is a collective call:
   AL_START covers the shard's own events, AL_LEVEL / AL_NANCHOR / AL_RESIDUAL and the result are
   job-wide (small all-gathers between the shards). Errors: SCAN_E_ORDER (no
   instances yet), SCAN_E_INVALID_ARG (no start_ns, reference out of range), SCAN_E_UNSUPPORTED
   (collective end times decrease along a rank's program order), SCAN_E_NCCL, SCAN_E_OOM,
   SCAN_E_CUDA.                                                                                  */
typedef struct scan_align_config { int32_t reference; uint32_t reserved; } scan_align_config;
typedef struct scan_align_result {
    uint64_t n_anchors;
    uint32_t n_aligned_ranks, n_unaligned_ranks, max_level, reserved;
    uint64_t max_residual_ns;
} scan_align_result;
scan_status scan_align(scan_ctx* ctx, const scan_align_config* cfg, scan_align_result* out);

/* ---- NEXT-3: sliding-window streaming ("on-line") -------------
   The context keeps the last `window_iters` pushed iterations. After every scan_stream_push the
   window-level outputs (RK_SUM_*, WD_*, WL_*, LK_*, LB_*, EG_*) equal scan_analyze on the
   window's events as one analysis window (the dcfg window_iters is ignored), but each push
   analyses only the new iteration: per-iteration partials are kept in a ring and recombined on
   the device (instances never straddle an iteration, reading R30; stage-2 segments crossing an
   iteration boundary are fixed up as between shards; link medians over the window's samples).
   scan_stream_open: topology + comm table of the job (copied), window length (1..4096), configs.
   scan_stream_push: `iteration` = the events of ONE whole iteration of every rank, the columns
   as for scan_load_events (HOST or DEVICE pointers, borrowed only for the call). Returns SCAN_OK
   or SCAN_PARTIAL (integrity reports in the window); out (optional) receives the window's
   verdict / walk counts. Errors: SCAN_E_ORDER (push before open), SCAN_E_UNSUPPORTED (an
   iteration is not SPMD, or its channel structure differs from the first one; sharded context),
   load errors of scan_load_events. Other outputs are unavailable on a stream context
   (SCAN_E_UNSUPPORTED). scan_stream_window: iterations currently in the window.               */
scan_status scan_stream_open(scan_ctx* ctx, const scan_topology* topo, const scan_comm_table* comms, uint32_t window_iters,
                             const scan_detect_config* dcfg, const scan_localize_config* lcfg);
scan_status scan_stream_push(scan_ctx* ctx, const scan_event_columns* iteration, uint32_t flags, scan_localize_result* out);
uint64_t    scan_stream_window(const scan_ctx* ctx);
scan_status scan_create_sharded(scan_ctx** out, int cuda_device, void* cuda_stream, int n_shards, int shard,
                                const uint8_t nccl_unique_id[128]);

/* In-process shard group (exchange back-end for testing and single-process use): n_shards (1..16)
   sharded contexts of ONE process, each driven by its own host thread, exchange through host barriers
   and device copies instead of NCCL; they may share a GPU. scan_create_sharded_local creates shard
   `shard` of `group` (same semantics and preconditions as scan_create_sharded). The group is owned by
   the caller and must outlive its contexts; scan_analyze on the shards must be called concurrently
   (one thread per shard), else it blocks. Not a performance path.                */
typedef struct scan_local_group scan_local_group;
scan_status scan_local_group_create(scan_local_group** out, int n_shards);
void scan_local_group_destroy(scan_local_group* group);
scan_status scan_create_sharded_local(scan_ctx** out, int cuda_device, void* cuda_stream, scan_local_group* group,
                                      int shard);

/* ---- NEXT-4: event-level blame (DESIGN.md §10e EB1-EB6) ----
   For every waiting communication event (an event of a VALID instance with wait > 0), the event
   where its delay began: it waited for the instance's last arriver, whose previous event in program
   order delayed it (EB2); a communication event that did not wait was itself delayed by its own
   previous event (EB3); compute events and the first event of a rank are roots. The pointers are
   followed to a root by pointer jumping on the device; a chain that never reaches a root (a pointer
   cycle, possible only in inconsistent traces) is unattributed (EB4). Each wait is blamed on the
   root's rank (EB5): BL_INFLICTED (on other ranks), BL_SELF, BL_UNATTRIBUTED, BL_SUFFERED; the
   whole loaded trace is one window (EB6). Requires a completed analysis (scan_analyze or
   scan_localize). On a sharded context (scan_create_sharded*) it is a collective call: each shard
   follows its chains locally, the chains that leave its iteration block are resolved over the
   earlier shards' per-rank tables (one all-gather), the per-rank sums are all-reduced, and
   BL_ROOT holds job-wide event ids (rank-major over the whole job) for the shard's own events;
   rounds / n_active are the shard's. Errors: SCAN_E_ORDER, SCAN_E_UNSUPPORTED (stream context,
   >= 2^32-16-world events per GPU), SCAN_E_NCCL, SCAN_E_OOM, SCAN_E_CUDA.                       */
typedef struct scan_blame_result {
    uint64_t n_waiting, n_cyclic;   /* waiting events; of them on a pointer cycle                     */
    uint64_t total_wait_ns;         /* sum of their waits                                             */
    uint32_t rounds;                /* pointer-jumping rounds                                         */
    uint32_t top_rank;              /* rank with the largest BL_INFLICTED (UINT32_MAX if none)        */
    uint64_t n_active;              /* events whose pointer is not a root (the jumping rounds' work)  */
} scan_blame_result;
scan_status scan_blame(scan_ctx* ctx, scan_blame_result* out);

/* ---- NEXT-2: Chrome-trace JSON ingest and merged emit (DESIGN.md §10d J1-J12) -----
   scan_ingest_json parses, ON THE DEVICE, one or more JSON documents: the per-rank files the
   tracer writes ("every rank has its own recorded event sequence as a JSON file") or a
   merged document. `bytes` holds the documents back to back, document i = [doc_offsets[i],
   doc_offsets[i+1]) (doc_offsets: HOST, n_docs+1 entries, monotone, doc_offsets[0] = 0,
   doc_offsets[n_docs] = n_bytes); `bytes` is HOST memory (copied H2D, pinned recommended) or,
   with SCAN_DEVICE_PTRS in flags, device memory of the ctx device (borrowed for the call).
   Schema (J1-J9): a document is {"traceEvents":[...], ...} or a bare array; an element with
   "ph":"X" is a trace event with "ts"/"dur" (microseconds, <= 3 decimals, converted exactly to
   ns), "pid" (rank < tp*pp*dp), "cat" (compute, all_reduce, all_gather, reduce_scatter,
   broadcast, send, recv) and optional "args": op, iter_end, mb, chunk, bwd, warmup (tracers.scope
   metadata), "group" (ascending participant ranks, required for collectives),
   "peer" (required for send/recv), "bytes" (payload). Other elements ("ph" != "X") are skipped.
   Events are put in program order per rank (ascending ts, ties by input position), every
   distinct group becomes a communicator, numbered in order of first use in that order. On
   success the context is loaded exactly as scan_load_events would load those columns (with
   start_ns), so every analysis call and export follows; SCAN_OUT_EV_* input columns are
   readable with scan_loaded_column().
   Errors: SCAN_E_SCHEMA with out->err_kind = SCAN_JSON_SYNTAX (malformed JSON; offset = first
   byte rejected) or SCAN_JSON_SCHEMA (out->err_field = SCAN_JF_*, offset = the '{' of the
   offending element, or of the document root for SCAN_JF_TRACE_EVENTS); a syntax error anywhere
   wins over any schema error, among schema errors the smallest offset wins (J11). SCAN_E_INVALID_ARG
   (offsets), SCAN_E_UNSUPPORTED (> 2^32-1 elements; a 64-bit group-hash collision), load errors.
   J10: the whole input is validated JSON (UTF-8 excepted); keys, "cat" and "ph" are compared as
   raw bytes.                                                                                   */
#define SCAN_JSON_OK      0
#define SCAN_JSON_SYNTAX  1
#define SCAN_JSON_SCHEMA  2
enum { SCAN_JF_TRACE_EVENTS = 1, SCAN_JF_EVENT, SCAN_JF_PH, SCAN_JF_TS, SCAN_JF_DUR, SCAN_JF_PID, SCAN_JF_CAT,
       SCAN_JF_ARGS, SCAN_JF_OP, SCAN_JF_ITER_END, SCAN_JF_MB, SCAN_JF_CHUNK, SCAN_JF_BWD, SCAN_JF_WARMUP,
       SCAN_JF_GROUP, SCAN_JF_PEER, SCAN_JF_BYTES };
typedef struct scan_json_result {
    uint64_t n_events;      /* trace events loaded                                               */
    uint64_t n_skipped;     /* event-array elements with "ph" != "X"                              */
    uint32_t n_comms;       /* distinct participant lists                                         */
    int32_t  err_kind;      /* SCAN_JSON_*                                                        */
    int32_t  err_field;     /* SCAN_JF_* of a schema error                                        */
    uint32_t reserved;
    uint64_t err_offset;    /* byte offset into `bytes`                                           */
} scan_json_result;
scan_status scan_ingest_json(scan_ctx* ctx, const scan_topology* topo, const uint8_t* bytes, uint64_t n_bytes,
                             const uint64_t* doc_offsets, uint32_t n_docs, uint32_t flags, scan_json_result* out);

/* The loaded event columns (any load path): 0 start_ns (i64; needs start times), 1 dur_ns (u32),
   2 kind_op (u16), 3 meta (u16), 4 comm (u32), 5 payload (u32), 6 rank_offsets (u64 [W+1]),
   7 comm offsets (u64), 8 comm members (u32). Copies into dst (host or device); *bytes = size.
   dst NULL: size only. Errors: SCAN_E_ORDER (nothing loaded), SCAN_E_INVALID_ARG.            */
scan_status scan_loaded_column(scan_ctx* ctx, int column, void* dst, uint64_t dst_bytes, int dst_is_device, uint64_t* bytes);

/* scan_emit_chrome writes the merged Chrome Tracing document of the loaded job (P:L119-125:
   "merges them-ordered by time-into a single JSON file"; pid = rank) with every communication
   event's matched instance id in args.related_sync_op. Byte format J12: events ordered
   by (timestamp, rank, program order), ts/dur in microseconds with exactly 3 decimals, args in
   the fixed order op, iter_end, mb, chunk, bwd, warmup, group | peer, bytes, related_sync_op,
   zero-valued metadata omitted. SCAN_EMIT_ALIGNED: timestamps of the last scan_align.
   The document is built on the device: a call with dst NULL builds it and returns its size in
   *n_bytes; a call with dst (host or device memory of dst_bytes >= *n_bytes) copies the document
   built for the current state (load / analysis / alignment), building it first if needed. Requires start_ns at load and a match (scan_match_collectives or
   scan_analyze); errors: SCAN_E_ORDER, SCAN_E_INVALID_ARG, SCAN_E_UNSUPPORTED (stream
   context), SCAN_E_OOM, SCAN_E_CUDA. On a sharded context (scan_create_sharded*) the document
   holds the shard's own events (its iteration block) with job-wide instance ids; the job's
   document is the shards' event lists merged by (ts, pid, shard order).                       */
#define SCAN_EMIT_ALIGNED 1u
scan_status scan_emit_chrome(scan_ctx* ctx, uint32_t flags, void* dst, uint64_t dst_bytes, int dst_is_device, uint64_t* n_bytes);

/* A0 ingest: validate sizes, place the columns on the device, build the comm tables.
   Per-event schema validation happens in scan_match_collectives (one pass).
   Errors: SCAN_E_INVALID_ARG (sizes, alignment, rank_order), SCAN_E_UNSUPPORTED
   (world > 65535 or n_comms + world^2 >= 2^32), SCAN_E_OOM, SCAN_E_CUDA.                    */
scan_status scan_load_events(scan_ctx* ctx, const scan_topology* topo, const scan_comm_table* comms,
                             const scan_event_columns* cols, uint32_t flags);

/* A1-A3: sequence numbers per (rank, channel), instance ids = base(channel) + k, completeness,
   integrity, per-instance dmin/dmax/last arriver, per-event wait, per-rank sums.
   Channels: communicators by id, then P2P (src,dst) pairs ascending (reading R2-R4).
   Returns SCAN_OK, SCAN_PARTIAL (reports present), SCAN_E_SCHEMA (first bad event in the
   message), SCAN_E_INTEGRITY (with SCAN_STRICT), SCAN_E_UNSUPPORTED (a rank touching more than
   256 channels, >2^32-1 instances), SCAN_E_ORDER (no load).                                   */
scan_status scan_match_collectives(scan_ctx* ctx, scan_match_result* out);

/* A4: stage 1 (leave-one-out lower median of the other DP peers, common op-id prefix).
   Requires a match (else SCAN_E_ORDER). cfg NULL = defaults.                                  */
scan_status scan_detect(scan_ctx* ctx, const scan_detect_config* cfg, scan_detect_result* out);

/* A5-A8: stage 2, stage 3, verdicts, wait-for edges, frontier walk. Uses the windows of the
   preceding scan_detect. Requires detect (else SCAN_E_ORDER). cfg NULL = defaults.            */
scan_status scan_localize(scan_ctx* ctx, const scan_localize_config* cfg, scan_localize_result* out);

/* A1-A8 in one call: equivalent to scan_match_collectives + scan_detect + scan_localize with the
   given configs (NULL = defaults) and the same outputs. When every pipeline-stage block of the
   trace is SPMD (equal per-rank event counts, same communicator roles; checked at load) it runs
   the fused stage-tile pass (K9): one streaming read of the event columns, every event
   verified against its stage template; if any event fails verification the call transparently
   reruns the general path, so results never depend on the SPMD assumption. Returns as
   scan_match_collectives. Any of the result pointers may be NULL.                              */
scan_status scan_analyze(scan_ctx* ctx, const scan_detect_config* dcfg, const scan_localize_config* lcfg,
                         scan_match_result* mres, scan_detect_result* dres, scan_localize_result* lres);
/* 1 if the last scan_analyze used the fused path, 0 if it ran the general path.                 */
int scan_used_fused(const scan_ctx* ctx);
/* Disable (1) / re-enable (0) the fused path for this context (testing / comparison).          */
scan_status scan_force_general(scan_ctx* ctx, int force);
/* Fused-kernel variant for the next scan_load_events: -1 automatic (the persistent TMA-fed stage
   kernel when TP divides 32, TP*DP <= 128 and every rank's first event index is a multiple of 4;
   else the transposed warp-per-position kernel when TP divides 32 and TP*DP <= 256; else the
   generic tile kernel), 0 generic, 1 transposed, 2 persistent where applicable (testing /
   comparison).                                                                                  */
scan_status scan_fused_variant(scan_ctx* ctx, int variant);

/* ---- result export ------------------------------------------------------------------------ */
typedef enum scan_output {
    /* per event, event order (expanded from the compact native layouts) */
    SCAN_OUT_EV_INST = 0,      /* u32, UINT32_MAX for compute events                   */
    SCAN_OUT_EV_WAIT,          /* u32 ns, 0 for compute events / invalid instances     */
    SCAN_OUT_EV_SLOW,          /* u8, 1 = stage-1 slow compute event                   */
    SCAN_OUT_EV_REF,           /* u32 ns, UINT32_MAX if not compared (needs want_ref)  */
    /* channels [n_channels] */
    SCAN_OUT_CH_KIND, SCAN_OUT_CH_A, SCAN_OUT_CH_B, SCAN_OUT_CH_NMEM, SCAN_OUT_CH_NMAX, SCAN_OUT_CH_NMIN,
    SCAN_OUT_CH_BASE,          /* u8 kind (0 coll, 1 p2p), u32 a (comm / src), u32 b (dst or MAX),
                                  u32 members, u32 max count, u32 min count, u64 first instance id */
    /* instances [n_instances] */
    SCAN_OUT_IN_CHANNEL, SCAN_OUT_IN_K, SCAN_OUT_IN_FLAGS, SCAN_OUT_IN_DMIN, SCAN_OUT_IN_DMAX,
    SCAN_OUT_IN_LAST, SCAN_OUT_IN_NPRESENT, SCAN_OUT_IN_PAYLOAD,
    /* per rank [world] */
    SCAN_OUT_RK_SUM_COMPUTE, SCAN_OUT_RK_SUM_WAIT, SCAN_OUT_RK_SUM_TRANSFER,   /* u64 ns */
    /* per peer class (tp,pp) [tp*pp], class = pp*tp_size + tp */
    SCAN_OUT_CL_J, SCAN_OUT_CL_MISMATCH,
    /* per (window, rank) [n_windows*world] */
    SCAN_OUT_WD_TOTAL, SCAN_OUT_WD_SLOW, SCAN_OUT_WD_CAND, SCAN_OUT_WD_FRAC,
    SCAN_OUT_WL_JOINED, SCAN_OUT_WL_LATE, SCAN_OUT_WL_LATE_FRAC, SCAN_OUT_WL_VERDICT, SCAN_OUT_WL_LINK_SLOW,
    /* per (window, P2P channel) [n_windows*n_p2p_channels] */
    SCAN_OUT_LK_WINDOW, SCAN_OUT_LK_SRC, SCAN_OUT_LK_DST, SCAN_OUT_LK_N, SCAN_OUT_LK_MED_PAYLOAD,
    SCAN_OUT_LK_MED_TRANSFER, SCAN_OUT_LK_USED_WARM, SCAN_OUT_LK_SLOW, SCAN_OUT_LK_DIR, SCAN_OUT_LK_ELIGIBLE,
    SCAN_OUT_LK_MED_BW,
    /* per (window, rank) labels */
    SCAN_OUT_LB_LABEL, SCAN_OUT_LB_ROOT_KIND, SCAN_OUT_LB_ROOT_RANK, SCAN_OUT_LB_ROOT_SRC, SCAN_OUT_LB_DEPTH,
    SCAN_OUT_LB_TOTAL_WAIT,
    /* wait-for edges, sorted by (window, waiter, waited-on) [n_edges] */
    SCAN_OUT_EG_WINDOW, SCAN_OUT_EG_SRC, SCAN_OUT_EG_DST, SCAN_OUT_EG_WEIGHT,
    /* native compact layouts (zero-copy via scan_output_device_ptr) */
    SCAN_OUT_COMM_INST,        /* u32 per comm event, ranks concatenated, program order       */
    SCAN_OUT_COMM_WAIT,        /* u32 per comm event                                          */
    SCAN_OUT_SLOW_BITS,        /* u32 words, per rank ceil(n_compute/32) words, bit j = slow  */
    /* shard view (per channel): this context's instances of channel c are the occurrences
       [CH_SHARD_K0[c], CH_SHARD_K0[c] + CH_SHARD_N[c]), i.e. instance ids CH_BASE[c] + k.
       Unsharded: K0 = 0, N = CH_NMAX.                                                          */
    SCAN_OUT_CH_SHARD_K0,      /* u64 */
    SCAN_OUT_CH_SHARD_N,       /* u32 */
    /* timeline alignment (scan_align) */
    SCAN_OUT_AL_START,         /* i64 per event: start on the reference rank's clock             */
    SCAN_OUT_AL_LEVEL,         /* i32 per rank: BFS level from the reference, -1 = not reached     */
    SCAN_OUT_AL_NANCHOR,       /* u32 per rank: anchors of its clock map                           */
    SCAN_OUT_AL_RESIDUAL,      /* u64 per rank: max (instance aligned end - own aligned end), ns   */
    /* event-level blame (scan_blame) */
    SCAN_OUT_BL_ROOT,          /* u64 per event: root event of a waiting event; 2^64-1 = not waiting,
                                  2^64-2 = on a pointer cycle (unattributed)                          */
    SCAN_OUT_BL_INFLICTED,     /* u64 per rank: wait (ns) of OTHER ranks' events rooted on this rank   */
    SCAN_OUT_BL_SELF,          /* u64 per rank: wait of its own events rooted on itself                */
    SCAN_OUT_BL_UNATTRIBUTED,  /* u64 per rank: wait of its own events on a pointer cycle              */
    SCAN_OUT_BL_SUFFERED,      /* u64 per rank: all wait of its waiting events                         */
    SCAN_OUT__COUNT
} scan_output;

/* Byte size of an output (0 if not yet computed). */
scan_status scan_output_size(scan_ctx* ctx, scan_output which, uint64_t* bytes);
/* Copy an output into dst (host or device memory of dst_bytes >= size). Export of the event-order
   arrays runs a (untimed) expansion kernel. */
scan_status scan_export(scan_ctx* ctx, scan_output which, void* dst, uint64_t dst_bytes, int dst_is_device);
/* Device pointer of a native compact output (SCAN_OUT_COMM_INST, _COMM_WAIT, _SLOW_BITS); NULL otherwise. */
const void* scan_output_device_ptr(scan_ctx* ctx, scan_output which);

/* Number of hot-path kernel launches issued by the last match+detect+localize sequence. */
uint64_t scan_kernel_launches(const scan_ctx* ctx);

/* Optional per-kernel timing with CUDA events recorded on the ctx stream around every launch
   (enable = 1), accumulated until scan_timing_reset(). scan_kernel_timing() returns the number of
   distinct kernels; for 0 <= i < that number it fills the kernel name (static string), total
   milliseconds and launch count. Timing adds one event pair per launch; keep it off for the
   headline number. */
scan_status scan_set_timing(scan_ctx* ctx, int enable);
void        scan_timing_reset(scan_ctx* ctx);
int         scan_kernel_timing(scan_ctx* ctx, int i, const char** name, double* total_ms, uint64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* MEGASCAN_SCAN_H */
