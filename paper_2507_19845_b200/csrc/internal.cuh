// internal.cuh — context, device buffers and warp utilities of the megascan CUDA library.
// Product code (sm_100a). Shares nothing with oracle/.
#pragma once

#include <cstdint>
#include <cstddef>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/megascan/scan.h"

namespace ms {

constexpr uint32_t NONE32 = 0xFFFFFFFFu;
constexpr int TILE_EV = 2048;   // events per warp tile (one rank, program order)
constexpr int KCAP = 32;        // distinct channels per warp tile (one per lane)
constexpr int RCAP = 256;       // distinct channels per rank
constexpr int PCAP = 32;        // distinct P2P peers per rank
constexpr int LINK_CAP = 16384; // samples per (window, link) held in shared memory for the median
// fused SPMD stage-tile path (K9)
constexpr int ROLES = 32;       // 0..15 collective roles (index in the rank's sorted comm list), 16..31 P2P roles
constexpr int CROLES = 16;
constexpr int FCOLS = ROLES + 4;  // per-tile pre-pass columns: roles, ncomp, ncomm, niter, cc_last
constexpr uint32_t NOT_SPMD = 32u;  // Counters.overflow bit: fused path not applicable

// Member slot record (uint4), one per member slot of every instance, in slot order
// (slot = slot_base(channel) + k * |members| + member; a P2P instance i has its send slot at
// p2p_slot0 + 2 (i - p2p_inst0) and its receive slot right after it):
//   x  the member event's duration (its wait is x - the instance's dmin, computed where it is needed)
//   y  fused path: the member event's index among its rank's comm events (k_xwait_scatter)
//   z  global iteration (bits 0-27) | kind (bits 28-30) | sender's warm-up flag (bit 31, P2P send slot)
//   w  P2P slots: payload bytes (k_stage leaves the event's position in its rank there and
//      k_cross_reduce gathers the payload)
// One 16-byte store per member instead of five scattered arrays: a P2P instance's two slots are one
// 32-byte sector.
constexpr uint32_t SLOT_IT_MASK = 0x0FFFFFFFu;
constexpr uint32_t SLOT_MAX_ITERS = 1u << 28;
__device__ __forceinline__ uint32_t slot_z(uint32_t it, uint32_t kind, uint32_t warm) {
  return it | ((kind & 7u) << 28) | (warm << 31);
}
__device__ __forceinline__ uint32_t slot_kind(uint32_t z) { return (z >> 28) & 7u; }

// Stage-3 sample key of a P2P instance (k_link_median): the f64 ratio payload / transfer as sortable
// bits (positive: bit order = value order; exactly rounded, so monotone in the exact ratio), bit 63 =
// warm-up flag; LK_NONE when the instance is not a sample (invalid, or transfer 0). Written by the
// instance reduction (k_cross_reduce / k_inst_reduce), the X3 unpack and the stream window.
constexpr unsigned long long LK_NONE = 0x7FFFFFFFFFFFFFFFull;  // a NaN pattern: no finite ratio has it
constexpr unsigned long long LK_WARM = 1ull << 63;
__device__ __forceinline__ unsigned long long ratio_key(uint32_t p, uint32_t t) {
  return (unsigned long long)__double_as_longlong((double)p / (double)t);
}
__device__ __forceinline__ unsigned long long lk_sample_key(uint32_t flags, uint32_t t, uint32_t p) {
  if (!(flags & SCAN_F_VALID) || t == 0) return LK_NONE;
  return ratio_key(p, t) | ((flags & SCAN_F_WARMUP) ? LK_WARM : 0ull);
}

// ----------------------------------------------------------------------------- device buffers
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) { cudaFree(p); p = nullptr; cap = 0; }
    size_t b = bytes ? bytes : 16;
    b = (b + 255) & ~size_t(255);
    cudaError_t e = cudaMalloc(&p, b);
    if (e == cudaSuccess) cap = b;
    return e;
  }
  void release() { if (p) cudaFree(p); p = nullptr; cap = 0; }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

// Device counters written by kernels, read back once per call.
struct Counters {
  unsigned long long bad_event;      // atomicMin, ~0 = none
  unsigned int bad_reason;
  unsigned int overflow;             // bit0 tile keys, bit1 rank keys, bit2 p2p peers, bit3 link samples, bit4 link count
  unsigned long long n_incomplete, n_kind_mismatch, n_payload_mismatch;
  unsigned long long n_p2p;          // P2P channels
  unsigned long long n_comm, n_comp; // totals
  unsigned int max_niter;            // max iter_end count over ranks
  unsigned int n_iters;              // max (iteration index of last event) + 1
  unsigned long long n_instances, n_slots, p2p_slot0, p2p_inst0;
  unsigned long long n_bits_words;
  unsigned int max_ncomp;
  unsigned int pad;
  unsigned long long n_compared, n_slow, n_candidates, n_class_mismatch;
  unsigned long long n_link_slow, n_roots, n_victims, n_unattributed;
  unsigned long long v_count[6];
  unsigned long long n_edges;
  unsigned long long n_xinst;
  unsigned int min_niter;            // min iter_end count over ranks (shard regularity check)
  unsigned int n_end_ranks;          // ranks whose last event ends an iteration
};

// one collective operation of a grouped exchange on the in-process back-end (xch.cu)
enum { XU8 = 0, XU32 = 1, XU64 = 2, XF64 = 3 };
struct XOp { int kind; const void* send; void* recv; size_t n; int type; int peer; };  // kind: 0 send, 1 recv, 2 all-reduce

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  uint64_t launches = 0;

  // topology / inputs
  int TP = 0, PP = 0, DP = 0, W = 0;
  uint32_t n_comms = 0;
  uint64_t N = 0;
  bool loaded = false, matched = false, detected = false, localized = false;
  uint32_t flags = 0;
  std::vector<uint64_t> h_rank_off;
  DevBuf own_dur, own_kind, own_meta, own_comm, own_pay;
  const uint32_t* d_dur = nullptr; const uint16_t* d_kind = nullptr; const uint16_t* d_meta = nullptr;
  const uint32_t* d_comm = nullptr; const uint32_t* d_pay = nullptr;
  const int64_t* d_start = nullptr;      // optional (timeline alignment only)
  DevBuf own_start;
  DevBuf rank_off;                 // u64 [W+1]
  DevBuf coff, cmem, ccls;         // comm table (u64, u32) + stage-2 class per comm (u8)
  DevBuf rcomm_off, rcomm;         // rank -> comms CSR (u32 offsets, u32)
  DevBuf nbc_off, nbc;             // rank -> collective neighbours CSR (u64 offsets, u32)
  uint64_t nnz_c = 0;
  // tiles
  uint64_t n_tiles = 0;
  DevBuf tile_rank, tile_order, tile_start, rank_tile0;  // u32, u64, u32 [W+1]
  std::vector<uint32_t> h_rank_tile0;

  // match workspaces
  DevBuf t_nkeys, t_keys, t_cnt, t_pref, t_ncomm, t_niter, t_last, t_commpre, t_iterpre, t_prevj;
  DevBuf r_nkeys, r_keys, r_cnt, r_ncomm, r_niter, r_ncomp, r_lastit;
  DevBuf r_comm_off, r_comp_off, r_bits_off;          // u64 [W+1]
  DevBuf bitmap, bitpre, bmsum;                        // P2P channel bitmap (u32 words) + word prefix + block sums
  uint64_t n_bm_words = 0;
  DevBuf counters;                                     // Counters
  Counters hc{};
  DevBuf ch_nmax, ch_nmin, ch_base, ch_slot, ch_nsend, ch_nrecv;   // channels
  uint64_t NCH = 0, n_p2p = 0, n_comm = 0, n_comp = 0, n_inst = 0, n_slots = 0, p2p_slot0 = 0, p2p_inst0 = 0;
  uint32_t NIT = 0;        // citer row length - 1 (max iter_end count)
  uint32_t n_iters = 0;
  DevBuf inst_c, wait_c;                 // per comm event
  DevBuf cdur, cop;                      // per compute event (rank-compacted)
  DevBuf slots;                          // SlotRec (uint4) per member slot, slot order
  DevBuf lk_key;                         // u64 per P2P instance: stage-3 sample key (lk_sample_key)
  DevBuf inst_rec;                       // uint4 per instance {dmin, dmax, last_rank, flags | cls<<8}
  DevBuf citer;                          // u32 [W][NIT+1]
  DevBuf nbp, nbp_n;                     // P2P neighbours per rank [W][PCAP]
  DevBuf rk_sum;                         // u64 [3][W]

  // detect
  scan_detect_config dcfg{};
  uint32_t NW = 1;
  DevBuf bits, cref, cl_J, cl_max, cl_min;
  DevBuf wd_total, wd_slow, wd_cand, wd_frac;
  uint32_t max_ncomp = 0;
  uint64_t n_bits_words = 0;

  // localize
  scan_localize_config lcfg{};
  DevBuf wl_joined, wl_late, wl_frac, wl_verdict, wl_link_slow;
  DevBuf ewc, ewp;                       // edge weights [NW][nnz_c], [NW][W*PCAP]
  DevBuf lk_n, lk_used, lk_medp, lk_medt, lk_bw, lk_slow, lk_dir, lk_elig;
  DevBuf lb_label, lb_rkind, lb_rrank, lb_rsrc, lb_depth, lb_twait;
  DevBuf scratch;                        // export scratch

  // fused SPMD path (K9): host-built role tables, template pre-pass, per-tile bases
  bool spmd = false;                     // every stage block is SPMD-compatible (checked at load)
  bool fused_used = false;               // results of the last analysis come from the fused path
  bool tiles_ready = false;              // general tile prefixes exist (needed by event-order exports)
  bool xwait_pending = false;            // fused: cross-stage waits still in slot order (k_xwait_scatter on export)
  bool partial_tail = false;             // fused_all stops before candidates / links / walk (streaming sub-analysis)
  bool stream_mode = false;              // window-level outputs of a sliding-window stream (stream.cu)
  void* stream_state = nullptr;          // StreamState (stream.cu), owned
  uint32_t FT = 0, FR = 0, n_ftiles = 0; // positions per fused tile, ranks per stage, fused tiles
  std::vector<uint32_t> h_st_tile0, h_st_npos;
  DevBuf st_tile0, st_npos, role_comm, role_slot, role_type, ncroles;
  DevBuf ft_cols, ft_base, ft_last, st_tot;   // pre-pass counts [FCOLS][tiles], scanned bases, last comm, stage totals
  DevBuf ft_posA, ft_posB, ft_posK;           // per template position packed info + template kind_op
  DevBuf p2p_rbase;                      // u32 [W][16]: instance base of the P2P channel behind each P2P role
  DevBuf dlate, dinfo;                   // deferred stage-2 positions (first comm position of a tile)
  bool rows_aligned = false, rows_aligned8 = false;
  bool force_general = false;
  bool fused_t = false;                  // transposed fused kernel (TP divides 32, R <= 256)
  bool use_stage = false;                // persistent TMA-fed fused kernel (k_stage.cu): aligned rows, R <= 128
  DevBuf ft_tbase;                       // [n_ftiles][40] tile-major bases / counts / stage (k_stage)
  DevBuf tmaps;                          // [PP][3] CUtensorMap (dur, comm, kind) of k_stage, built on first use per load
  uint64_t load_id = 0, tmap_load = ~0ull; // scan_load_events counter; load the maps were built for
  bool kind2d = false;                   // kind rows of every stage 16-byte aligned with a 16-byte stride (2-D TMA)
  int fused_variant = -1;                // testing: -1 auto, 0 generic fused, 1 transposed, 2 persistent (k_stage)
  uint32_t NCRM = 1;                     // max collective roles of a rank over the stages
  DevBuf eidx;                           // [W][TP+DP] edge slot of each TP-/DP-group partner
  DevBuf tile_stage;                     // [n_ftiles] stage of each fused tile (u8)
  DevBuf xbase;                          // [NCH+1] cross-stage instance index
  DevBuf p2p_eslot;                      // [n_p2p][2] wait-for edge column per P2P link direction
  DevBuf xe_off, xe_col;                 // cross collectives: member x member edge-column tables (built at load)
  DevBuf xbig; uint32_t n_big = 0;       // cross collectives with more than 32 members (k_cross_big)
  uint64_t n_xinst = 0;
  // multi-GPU iteration-window shards (row A9, shard.cu); n_shards == 1: unsharded
  int n_shards = 1, shard = 0;
  void* nccl = nullptr;                  // ncclComm_t owned by the context
  void* lgroup = nullptr;                // in-process exchange group (xch.cu), not owned; nccl == nullptr then
  std::vector<XOp> xops;                 // pending ops of an in-process grouped exchange
  DevBuf xtmp;                           // in-process all-reduce scratch
  uint32_t it_off = 0;                   // global iteration of this shard's first iteration
  DevBuf g_base, g_slot, g_nmax, g_nmin, g_k0; // global channel tables + this shard's first occurrence per channel; (kernels use the shard-shifted ch_base/ch_slot)
  std::vector<uint64_t> h_shard_k0;      // [NCH] global occurrence index of this shard's first instance
  std::vector<uint32_t> h_shard_n;       // [NCH] this shard's instance count per channel
  std::vector<uint8_t> h_ccls;           // host copy of the stage-2 class per comm
  std::vector<uint64_t> h_coff;          // host copy of the comm offsets
  std::vector<uint32_t> h_cmem, h_rcomm, h_rcomm_off;  // host copies: comm members, rank -> comms CSR
  // timeline alignment (k_align.cu)
  bool aligned = false;
  DevBuf al_tend, al_aend, al_anct, al_anco, al_level, al_nanc, al_resid, al_flag, al_start, al_ranks, al_tgt;
  uint64_t g_N = 0, g_ncomm = 0, g_ncomp = 0;  // job-wide totals (sharded)
  DevBuf x_send, x_recv, x_recv2, x_ep, x_stage, headtail, lk_sendmap, lk_recvmap;
  void* h_pin = nullptr;                 // pinned host scratch (exchange read-backs, table staging)
  void* h_e = nullptr;                   // pinned: the X4 status words (checked after the final read-back)
  size_t h_pin_cap = 0;
  cudaEvent_t ev_x1 = nullptr, ev_x2 = nullptr;
  // event-level blame (k_blame.cu)
  bool blamed = false;
  DevBuf al_xs, al_xr, al_row, al_lt, al_init, al_bx, al_bnd, bl_xs, bl_xr, bl_gbase, bl_ext, al_imax, al_vbits, al_seg, bl_seg, bl_inst, bl_pa, bl_pb, bl_root, bl_last, bl_rank, bl_rk;
  // JSON ingest / emit state (k_json.cu), owned; gen: bumped by every load / analysis / alignment
  void* json_state = nullptr;
  uint64_t gen = 0;
  // queued zero / byte fills, flushed as one k_fill launch before the next kernel (flush_fills)
  struct Fill { void* p; uint64_t n; uint32_t v; };
  std::vector<Fill> fills;
  // optional per-kernel timing
  bool timing = false;
  struct Pending { int k; cudaEvent_t a, b; };
  std::vector<Pending> pend;
  std::vector<std::string> knames;
  std::vector<double> kms;
  std::vector<uint64_t> kcnt;
  std::vector<cudaEvent_t> evpool;

  bool fail(scan_status, const std::string& m) { err = m; return false; }
};

// queued buffer fills (instead of one cudaMemsetAsync API call each): every queued fill runs, in
// queue order, before the next kernel launched through timed() or after an explicit flush_fills()
inline void queue_fill(Ctx& c, void* p, uint64_t bytes, uint8_t v) { if (p && bytes) c.fills.push_back({p, bytes, v}); }
int flush_fills(Ctx& c);

// Launch wrapper: records an event pair around a launcher when timing is on.
bool sync_check_on();  // MS_SYNC_CHECK=1: synchronise after every launcher and name the one that faulted (diagnostics)
void sync_check(Ctx& c, const char* name);
template <class F>
int timed(Ctx& c, const char* name, F&& f) {
  flush_fills(c);
  if (sync_check_on()) { const int n = f(); sync_check(c, name); return n; }
  if (!c.timing) return f();
  int k = -1;
  for (size_t i = 0; i < c.knames.size(); ++i) if (c.knames[i] == name) k = (int)i;
  if (k < 0) { c.knames.push_back(name); c.kms.push_back(0); c.kcnt.push_back(0); k = (int)c.knames.size() - 1; }
  cudaEvent_t a, b;
  if (c.evpool.size() >= 2) { a = c.evpool.back(); c.evpool.pop_back(); b = c.evpool.back(); c.evpool.pop_back(); }
  else { cudaEventCreate(&a); cudaEventCreate(&b); }
  cudaEventRecord(a, c.stream);
  int n = f();
  cudaEventRecord(b, c.stream);
  c.pend.push_back({k, a, b});
  return n;
}
void resolve_timing(Ctx& c);

// CUDA error -> scan_status with the message in c.err (host orchestration code; needs `Ctx& c`)
#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t _e = (x);                                                              \
    if (_e != cudaSuccess) {                                                           \
      c.err = std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " #x;        \
      return _e == cudaErrorMemoryAllocation ? SCAN_E_OOM : SCAN_E_CUDA;               \
    }                                                                                  \
  } while (0)

// read back the device counters (synchronises the context stream)
scan_status sync_read(Ctx& c);
template <class T>
scan_status upload(Ctx& c, DevBuf& b, const std::vector<T>& v) {
  CK(b.ensure(v.size() * sizeof(T)));
  if (!v.empty()) CK(cudaMemcpyAsync(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, c.stream));
  return SCAN_OK;
}
// host orchestration shared by the single-GPU paths (api.cu) and the shard path (shard.cu)
scan_status prep_ws(Ctx& c, bool tiles);
scan_status alloc_match_buffers(Ctx& c, bool fused);
scan_status alloc_detect(Ctx& c);
scan_status alloc_localize(Ctx& c);
scan_status sharded_all(Ctx& c);
scan_status fused_all(Ctx& c);
scan_status fused_rerun(Ctx& c);
int launch_shard_head(Ctx& c, unsigned long long* out);
// exchange layer of the sharded analysis (xch.cu): NCCL communicator or in-process group; 0 = ok
int xch_allgather(Ctx& c, const void* send, void* recv, size_t n_u32);
void xch_group_start(Ctx& c);
void xch_send(Ctx& c, const void* p, size_t n_u32, int peer);
void xch_recv(Ctx& c, void* p, size_t n_u32, int peer);
void xch_allreduce(Ctx& c, void* p, size_t n, int type);
int xch_group_end(Ctx& c);
const char* xch_error(int rc);
int launch_shard_fixup(Ctx& c, int G, const unsigned long long* ht);
int launch_link_median_window(Ctx& c, const uint64_t* base, const uint32_t* nmax, const uint64_t* slot, const uint4* rec,
                              const uint32_t* iter, const uint32_t* pay, const unsigned long long* key, uint64_t n_inst);
scan_status align_all(Ctx& c, int32_t ref, scan_align_result* out);
scan_status ensure_tiles(Ctx& c);
void shard_release(Ctx& c);
void stream_release(Ctx& c);
void json_release(Ctx& c);
scan_status blame_all(Ctx& c, scan_blame_result* out);

}  // namespace ms

struct scan_ctx { ms::Ctx c; };  // the opaque handle of scan.h

namespace ms {

// ----------------------------------------------------------------------------- device helpers
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xFFFFFFFFu, v, o);
    if (lane_id() >= (uint32_t)o) v += t;
  }
  return v;
}
__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, uint32_t& total) {
  uint32_t inc = warp_incl_scan(v);
  total = __shfl_sync(0xFFFFFFFFu, inc, 31);
  return inc - v;
}
__device__ __forceinline__ int32_t warp_incl_max(int32_t v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t t = __shfl_up_sync(0xFFFFFFFFu, v, o);
    if (lane_id() >= (uint32_t)o) v = max(v, t);
  }
  return v;
}
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}
__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
  return __reduce_add_sync(0xFFFFFFFFu, v);
}

// 8 consecutive events starting at group index g (multiple of 8) — vectorised when in bounds.
__device__ __forceinline__ void load8_u16(const uint16_t* __restrict__ p, uint64_t g, uint64_t n, uint16_t out[8]) {
  if (g + 8 <= n) {
    uint4 v = __ldg(reinterpret_cast<const uint4*>(p + g));
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int s = 0; s < 8; ++s) out[s] = (uint16_t)(w[s >> 1] >> ((s & 1) * 16));
  } else {
#pragma unroll
    for (int s = 0; s < 8; ++s) out[s] = (g + s < n) ? p[g + s] : 0;
  }
}
__device__ __forceinline__ void load8_u32(const uint32_t* __restrict__ p, uint64_t g, uint64_t n, uint32_t out[8]) {
  if (g + 8 <= n) {
    uint4 a = __ldg(reinterpret_cast<const uint4*>(p + g));
    uint4 b = __ldg(reinterpret_cast<const uint4*>(p + g + 4));
    out[0] = a.x; out[1] = a.y; out[2] = a.z; out[3] = a.w;
    out[4] = b.x; out[5] = b.y; out[6] = b.z; out[7] = b.w;
  } else {
#pragma unroll
    for (int s = 0; s < 8; ++s) out[s] = (g + s < n) ? p[g + s] : 0;
  }
}

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t n, uint32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) { uint32_t m = (lo + hi) >> 1; if (a[m] < x) lo = m + 1; else hi = m; }
  return lo;
}
// index of the last element <= x in a sorted u64 array of length n (a[0] <= x assumed)
__device__ __forceinline__ uint64_t upper_bound_u64(const uint64_t* a, uint64_t n, uint64_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) { uint64_t m = (lo + hi) >> 1; if (a[m] <= x) lo = m + 1; else hi = m; }
  return lo;
}

// exact ratio order p_a/t_a < p_b/t_b  (t > 0)
__device__ __forceinline__ bool ratio_less(uint32_t pa, uint32_t ta, uint32_t pb, uint32_t tb) {
  return (unsigned long long)pa * tb < (unsigned long long)pb * ta;
}

// ----------------------------------------------------------------------------- block scans
template <int NT>
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t v, uint32_t& total, uint32_t* sm /*[32]*/) {
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
  uint32_t inc = warp_incl_scan(v);
  if (lane == 31) sm[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    uint32_t x = lane < NT / 32 ? sm[lane] : 0;
    uint32_t xi = warp_incl_scan(x);
    sm[lane] = xi - x;
    if (lane == 31) sm[32] = xi;
  }
  __syncthreads();
  uint32_t r = sm[wid] + inc - v;
  total = sm[32];
  __syncthreads();
  return r;
}
template <int NT>
__device__ __forceinline__ int32_t block_excl_max(int32_t v, int32_t& total, int32_t* sm /*[33]*/) {
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
  int32_t inc = warp_incl_max(v);
  int32_t ex = __shfl_up_sync(0xFFFFFFFFu, inc, 1);
  if (lane == 0) ex = INT32_MIN;
  if (lane == 31) sm[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int32_t x = lane < NT / 32 ? sm[lane] : INT32_MIN;
    int32_t xi = warp_incl_max(x);
    int32_t xe = __shfl_up_sync(0xFFFFFFFFu, xi, 1);
    sm[lane] = lane == 0 ? INT32_MIN : xe;
    if (lane == 31) sm[32] = xi;
  }
  __syncthreads();
  int32_t r = max(sm[wid], ex);
  total = sm[32];
  __syncthreads();
  return r;
}

// ----------------------------------------------------------------------------- kernel launchers
// (each returns the number of kernel launches it enqueued)
int launch_tile_scan(Ctx& c);
int launch_rank_scan(Ctx& c);
int launch_rank_prefix(Ctx& c);
int launch_p2p_channels(Ctx& c);
int launch_assign(Ctx& c);
int launch_inst_reduce(Ctx& c);
int launch_stage1(Ctx& c);
int launch_class_counts(Ctx& c);
int launch_stage1_counts(Ctx& c);
int launch_event_pass(Ctx& c);
int launch_links(Ctx& c);
int launch_link_median(Ctx& c);
int launch_link_flags(Ctx& c);
int launch_p2p_counts(Ctx& c);
int launch_p2p_counts_to(Ctx& c, uint32_t* nsend, uint32_t* nrecv, uint32_t* psrc, uint32_t* pdst);
int launch_verdict_walk(Ctx& c);
// exports
int launch_expand_events(Ctx& c, scan_output which, void* dst);
int launch_instance_export(Ctx& c, scan_output which, void* dst);
// fused path
int launch_fused_prepass(Ctx& c);
int launch_fused_census(Ctx& c);
int launch_fused(Ctx& c);
bool p2p_defer_on(Ctx& c);
// general-path tile kernels walk the tiles interleaved across ranks (Ctx::tile_order) unless
// MS_TILE_ORDER=0 (index order, rank-major)
const uint32_t* tile_order_ptr(Ctx& c);
int launch_p2p_roles(Ctx& c);
int launch_stage(Ctx& c);
// the analysis runs k_stage: selected at load and the channel bases fit its 32-bit tables
inline bool stage_active(const Ctx& c) { return c.use_stage && c.n_inst < (1ull << 32) && c.n_slots < (1ull << 32); }
uint32_t stage_tile(uint32_t R, uint32_t TP, uint32_t DP, uint32_t NCRM, uint32_t PP);
size_t fused_smem_bytes(uint32_t T, uint32_t R, uint32_t TP, uint32_t DP, uint32_t NCRM);
size_t fused_t_smem_bytes(uint32_t T, uint32_t R, uint32_t TP, uint32_t DP, uint32_t NCRM);
size_t fused_t_smem_cap();
uint32_t fused_t_tile_events();
int launch_cross_reduce(Ctx& c);
int launch_xwait_scatter(Ctx& c);
int launch_deferred(Ctx& c);
int launch_wd_finish(Ctx& c);

}  // namespace ms
