// k_blame.cu — NEXT-4: event-level blame by pointer jumping (readings EB1-EB6).
//
// The paper's insight: ranks that suffer collateral slowdown "only lag because they are
// waiting for the faulty peer". Every waiting communication event (valid instance, wait > 0) points
// at the event that delayed the instance's last arriver (that rank's previous event); a communication
// event that did not wait points at its own rank's previous event; compute events and the first
// event of a rank are roots. Following the pointers gives, for every wait, the event where the delay
// began; pointer jumping (ptr <- ptr[ptr]) resolves all chains in log2(longest chain) rounds.
//   k_bl_last   per instance: where its waiting members point -- the previous event of its last
//               arriver's member event (that event itself if it is its rank's first)   (tile warps)
//   k_bl_ptr    per event: the pointer (u32 event index)                      (tile warps)
//   k_bl_jump0 / k_bl_jumpk  one jumping round (in place; round 1 over every event, later rounds over the
//               per-block lists of pointers that moved), with a change flag
//   k_bl_sum    terminal check (a fixed point of the ORIGINAL pointers; anything else is a cycle),
//               per-event root, per-rank inflicted / self / unattributed / suffered wait
#include "internal.cuh"

namespace ms {
namespace {

constexpr unsigned long long BL_NONE = ~0ull, BL_CYCLE = ~0ull - 1;

struct BA {
  uint64_t n_tiles;
  const uint32_t* tile_rank; const uint64_t* tile_start; const uint64_t* rank_off;
  // per comm event, comm order (inst_c / wait_c): event x of tile t is comm event
  // comm_off[rank] + t_commpre[t] + (comm events of the tile before x)
  const uint16_t* kind; const uint32_t* inst; const uint32_t* wait; const uint4* rec;
  const uint64_t* comm_off; const uint32_t* t_commpre;
  uint32_t* last_ev;  // per instance: the pointer target of its waiting members (EB2)
  uint32_t* ptr0;    // unused (null)
  uint16_t* rank16;  // per event: its rank if the event is a root of the ORIGINAL pointers, else 0xFFFF
  uint32_t* ptr; unsigned int* n_active;  // working pointers (jumped in place), events that are not roots
  // sharded context, shard > 0: a rank's first local event is not its job-wide first one; what precedes
  // it is the rank's last event on the previous shard, pointer value N + rank (resolved across shards)
  uint32_t ext; uint64_t N;
  const uint32_t* order;  // processing order of the tiles (tile_order_ptr), null = index order
};

// A communication event waited iff its wait is > 0 (EB1): the wait is 0 for every member of an
// invalid instance, and the last arriver of a valid one waits 0, so only events with wait 0 can be the
// last arriver's member and need the instance record.
__global__ void __launch_bounds__(256) k_bl_last(BA a) {
  uint64_t tile = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (tile >= a.n_tiles) return;
  if (a.order) tile = a.order[tile];
  const uint32_t r = a.tile_rank[tile];
  const uint64_t rs = a.rank_off[r];
  const uint64_t s = a.tile_start[tile], e = min(s + (uint64_t)TILE_EV, a.rank_off[r + 1]);
  const uint32_t lane = lane_id();
  uint64_t ci0 = a.comm_off[r] + a.t_commpre[tile];  // comm index of the chunk's first comm event
  for (uint64_t x0 = s; x0 < e; x0 += 32) {
    const uint64_t x = x0 + lane;
    const bool isc = x < e && (a.kind[x] & 7u) != 0;
    const unsigned bm = __ballot_sync(0xFFFFFFFFu, isc);
    const uint64_t ci = ci0 + __popc(bm & ((1u << lane) - 1u));
    ci0 += __popc(bm);
    if (!isc || a.wait[ci] != 0) continue;
    const uint32_t I = a.inst[ci];
    const uint4 rc = a.rec[I];
    if ((rc.w & SCAN_F_VALID) && rc.z == r) a.last_ev[I] = (uint32_t)(x != rs ? x - 1 : (a.ext ? a.N + r : x));
  }
}

__global__ void __launch_bounds__(256) k_bl_ptr(BA a) {
  __shared__ unsigned int blk_act;
  if (threadIdx.x == 0) blk_act = 0;
  __syncthreads();
  uint64_t tile = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  uint32_t n_act = 0;
  if (tile < a.n_tiles) {
    if (a.order) tile = a.order[tile];
    const uint32_t r = a.tile_rank[tile];
    const uint64_t rs = a.rank_off[r];
    const uint64_t s = a.tile_start[tile], e = min(s + (uint64_t)TILE_EV, a.rank_off[r + 1]);
    constexpr int U = 4;  // 4 x 32 events per step, every step's loads issued before they are used
    const uint32_t lane = lane_id();
    uint64_t ci0 = a.comm_off[r] + a.t_commpre[tile];
    for (uint64_t xb = s; xb < e; xb += 32 * U) {  // warp-uniform bound (ballots below)
      const uint64_t x0 = xb + lane;
      uint16_t ko[U];
      uint32_t wt[U], in[U];
      uint64_t ci[U];
#pragma unroll
      for (int u = 0; u < U; ++u) { const uint64_t x = x0 + 32u * u; ko[u] = x < e ? a.kind[x] : (uint16_t)0; }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned bm = __ballot_sync(0xFFFFFFFFu, (ko[u] & 7u) != 0);
        ci[u] = ci0 + __popc(bm & ((1u << lane) - 1u));
        ci0 += __popc(bm);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) wt[u] = (ko[u] & 7u) ? a.wait[ci[u]] : 0u;
#pragma unroll
      for (int u = 0; u < U; ++u) in[u] = wt[u] > 0 ? a.inst[ci[u]] : 0u;
#pragma unroll
      for (int u = 0; u < U; ++u) in[u] = wt[u] > 0 ? a.last_ev[in[u]] : 0u;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t x = x0 + 32u * u;
        if (x >= e) break;
        uint64_t p;
        if ((ko[u] & 7u) == 0) p = x;       // EB3: compute events are roots
        else if (wt[u] > 0) p = in[u];      // EB2: the last arriver's previous event
        else p = x != rs ? x - 1 : (a.ext ? a.N + r : x);  // EB3: own previous event
        a.ptr[x] = (uint32_t)p;
        a.rank16[x] = p == x ? (uint16_t)r : (uint16_t)0xFFFFu;  // W <= 65535: 0xFFFF is no rank
        n_act += p != x;
      }
    }
  }
  n_act = warp_sum_u32(n_act);
  if (lane_id() == 0 && n_act) atomicAdd(&blk_act, n_act);
  __syncthreads();
  if (threadIdx.x == 0 && blk_act) atomicAdd(a.n_active, blk_act);  // one global atomic per block
}

// Pointer jumping on compacted lists: round 1 visits every event; an event whose pointer moved stays
// on its block's list for the next round (the others have reached a root, or will be found there next
// round and dropped), so later rounds cost only what is still moving. Lists are segmented per block
// (block b owns [b S, (b+1) S) of each list buffer): no global counter, no atomics on the append.
constexpr int JB_NT = 256;

// block-level append of the flagged threads' x to out[nout ...]; nout is block-uniform
__device__ __forceinline__ void jb_append(bool act, uint32_t x, uint32_t* out, uint32_t& nout, uint32_t* wcnt) {
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
  const unsigned bm = __ballot_sync(0xFFFFFFFFu, act);
  if (lane == 0) wcnt[wid] = (uint32_t)__popc(bm);
  __syncthreads();
  uint32_t off = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < JB_NT / 32; ++w) { const uint32_t v = wcnt[w]; off += (w < (int)wid) ? v : 0u; tot += v; }
  if (act) out[nout + off + __popc(bm & ((1u << lane) - 1u))] = x;
  __syncthreads();  // wcnt is reused by the next call
  nout += tot;
}

__device__ __forceinline__ bool jb_step(uint32_t* ptr, uint32_t x, uint64_t N) {
  const uint32_t p = ptr[x];
  if (p == x || p >= N) return false;  // a root, or a rank's entry from the previous shard (terminal here)
  const uint32_t q = ptr[p];
  if (q == p) return false;
  ptr[x] = q;
  return true;
}

__global__ void __launch_bounds__(JB_NT) k_bl_jump0(uint64_t N, uint64_t S, uint32_t* ptr, uint32_t* list_out, uint32_t* seg_out,
                                                    unsigned int* changed) {
  __shared__ uint32_t wcnt[JB_NT / 32];
  uint32_t* out = list_out + (uint64_t)blockIdx.x * S;
  uint32_t nout = 0;
  for (uint64_t c0 = (uint64_t)blockIdx.x * JB_NT; c0 < N; c0 += (uint64_t)gridDim.x * JB_NT) {
    const uint64_t x = c0 + threadIdx.x;
    const bool act = x < N && jb_step(ptr, (uint32_t)x, N);
    jb_append(act, (uint32_t)x, out, nout, wcnt);
  }
  if (threadIdx.x == 0) { seg_out[blockIdx.x] = nout; if (nout) atomicOr(changed, 1u); }
}

__global__ void __launch_bounds__(JB_NT) k_bl_jumpk(uint64_t N, uint64_t S, uint32_t* ptr, const uint32_t* list_in,
                                                    const uint32_t* seg_in, uint32_t* list_out, uint32_t* seg_out,
                                                    unsigned int* changed) {
  __shared__ uint32_t wcnt[JB_NT / 32];
  const uint32_t nin = seg_in[blockIdx.x];
  const uint32_t* in = list_in + (uint64_t)blockIdx.x * S;
  uint32_t* out = list_out + (uint64_t)blockIdx.x * S;
  uint32_t nout = 0;
  for (uint32_t i0 = 0; i0 < nin; i0 += JB_NT) {
    const uint32_t i = i0 + threadIdx.x;
    uint32_t x = 0;
    bool act = false;
    if (i < nin) { x = in[i]; act = jb_step(ptr, x, N); }
    jb_append(act, x, out, nout, wcnt);
  }
  if (threadIdx.x == 0) { seg_out[blockIdx.x] = nout; if (nout) atomicOr(changed, 1u); }
}

struct SA {
  BA b; uint32_t W; const uint32_t* ptr; unsigned long long* root;
  unsigned long long* inflicted; unsigned long long* self_; unsigned long long* unattr; unsigned long long* suffered;
  unsigned long long* counts;  // [0] waiting events, [1] on a cycle
  int smem_hist;               // 1: inflicted wait accumulated in a shared-memory histogram over ranks
  // sharded: job-wide event id of local event p of rank q = gbase[q] + p; ext[r] = the resolved root of
  // pointer N + r: {id lo, id hi, rank, 1 = root / 0 = on a cycle}
  const unsigned long long* gbase; const uint4* ext;
};

// Persistent over tiles (one warp per tile). Most waits of a job root on a few ranks, so the inflicted
// wait goes through a block-local shared-memory histogram (one global atomic per block and rank);
// same-address global atomics would serialise in L2.
#ifndef MS_BS_MINB
#define MS_BS_MINB 4  // one resident wave of 4 CTAs per SM (6 per SM measured slower: 9.7 -> 11.0 ms)
#endif
__global__ void __launch_bounds__(256, MS_BS_MINB) k_bl_sum(SA a) {
  extern __shared__ unsigned long long sh_inf[];
  if (a.smem_hist) {
    for (uint32_t i = threadIdx.x; i < a.W; i += blockDim.x) sh_inf[i] = 0;
    __syncthreads();
  }
  unsigned long long nw = 0, ncy = 0;
  for (uint64_t ti = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5); ti < a.b.n_tiles; ti += (uint64_t)gridDim.x * 8) {
    const uint64_t tile = a.b.order ? a.b.order[ti] : ti;
    const uint32_t r = a.b.tile_rank[tile];
    const uint64_t s = a.b.tile_start[tile], e = min(s + (uint64_t)TILE_EV, a.b.rank_off[r + 1]);
    unsigned long long suf = 0, slf = 0, una = 0;
    uint32_t run_r = 0xFFFFFFFFu;  // per-lane run of inflicted wait on one rank
    unsigned long long run_w = 0;
    constexpr int U = 4;  // 4 x 32 events per step, the loads of a step issued together
    const uint32_t lane = lane_id();
    uint64_t ci0 = a.b.comm_off[r] + a.b.t_commpre[tile];
    for (uint64_t base = s; base < e; base += 32 * U) {
      uint32_t wv[U], pv[U], rv[U];
      uint16_t ko[U];
      uint64_t ci[U];
#pragma unroll
      for (int u = 0; u < U; ++u) { const uint64_t x = base + 32u * u + lane; ko[u] = x < e ? a.b.kind[x] : (uint16_t)0; }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned bm = __ballot_sync(0xFFFFFFFFu, (ko[u] & 7u) != 0);
        ci[u] = ci0 + __popc(bm & ((1u << lane) - 1u));
        ci0 += __popc(bm);
      }
      // the comm events' waits (comm order); compute events wait 0
#pragma unroll
      for (int u = 0; u < U; ++u) wv[u] = (ko[u] & 7u) ? a.b.wait[ci[u]] : 0u;
#pragma unroll
      for (int u = 0; u < U; ++u) pv[u] = wv[u] ? a.ptr[base + 32u * u + lane_id()] : 0u;
#pragma unroll
      for (int u = 0; u < U; ++u) rv[u] = (wv[u] && pv[u] < a.b.N) ? (uint32_t)a.b.rank16[pv[u]] : 0xFFFFu;
#pragma unroll
      for (int u = 0; u < U; ++u) {
      const uint64_t x = base + 32u * u + lane_id();
      if (x >= e) break;
      const unsigned long long w = wv[u];  // EV_WAIT: 0 for compute events and invalid instances
      unsigned long long root = BL_NONE;
      if (w) {
        const uint32_t p = pv[u];
        ++nw;
        suf += w;
        uint32_t rr = rv[u];  // one gather: the root's rank, or 0xFFFF (not a root: a cycle)
        unsigned long long rid = p;
        if (p >= a.b.N) {  // the chain left the shard: its root, resolved on the earlier shards
          const uint4 xe = a.ext[p - a.b.N];
          rr = xe.w ? xe.z : 0xFFFFu;
          rid = (unsigned long long)xe.y << 32 | xe.x;
        } else if (a.gbase && rr != 0xFFFFu) {
          rid = a.gbase[rr] + p;
        }
        if (rr != 0xFFFFu) {  // a root of the original pointers
          root = rid;
          if (rr == r) slf += w;
          else {
            if (rr != run_r) {
              if (run_w) { if (a.smem_hist) atomicAdd(&sh_inf[run_r], run_w); else atomicAdd(&a.inflicted[run_r], run_w); }
              run_r = rr; run_w = 0;
            }
            run_w += w;
          }
        } else {
          root = BL_CYCLE;
          una += w;
          ++ncy;
        }
      }
      a.root[x] = root;
      }
    }
    if (run_w) { if (a.smem_hist) atomicAdd(&sh_inf[run_r], run_w); else atomicAdd(&a.inflicted[run_r], run_w); }
    suf = warp_sum_u64(suf); slf = warp_sum_u64(slf); una = warp_sum_u64(una);
    if (lane_id() == 0) {
      if (suf) atomicAdd(&a.suffered[r], suf);
      if (slf) atomicAdd(&a.self_[r], slf);
      if (una) atomicAdd(&a.unattr[r], una);
    }
  }
  nw = warp_sum_u64(nw); ncy = warp_sum_u64(ncy);
  if (lane_id() == 0) {
    if (nw) atomicAdd(&a.counts[0], nw);
    if (ncy) atomicAdd(&a.counts[1], ncy);
  }
  if (a.smem_hist) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < a.W; i += blockDim.x)
      if (sh_inf[i]) atomicAdd(&a.inflicted[i], sh_inf[i]);
  }
}

inline unsigned nbk(uint64_t n, unsigned t) { return (unsigned)std::max<uint64_t>(1, (n + t - 1) / t); }

// Sharded blame: what the LAST local event of every rank resolves to after the local jumping, one row
// of the all-gather: [4 r + 0..3] = {0 root: root rank, its offset within that rank's local events | 1
// the rank's entry from the previous shard: rank | 2 on a cycle}, then [4 W + r] = local event count.
// A rank without local events passes its entry through (type 1, itself).
__global__ void k_bl_ltab(uint32_t W, uint64_t N, const uint64_t* rank_off, const uint32_t* ptr, const uint16_t* rank16,
                          uint32_t* row) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= W) return;
  const uint64_t b = rank_off[r], e = rank_off[r + 1];
  uint32_t t = 1, v = r, k = 0;
  if (e > b) {
    const uint32_t p = ptr[e - 1];
    if (p >= N) { t = 1; v = (uint32_t)(p - N); }
    else if (rank16[p] != 0xFFFFu) { t = 0; v = rank16[p]; k = (uint32_t)(p - rank_off[rank16[p]]); }
    else { t = 2; v = 0; }
  }
  row[4 * r] = t; row[4 * r + 1] = v; row[4 * r + 2] = k; row[4 * r + 3] = 0;
  row[4 * W + r] = (uint32_t)(e - b);
}

// Sharded blame (collective): exchange every shard's per-rank table (k_bl_ltab) and resolve, for this
// shard, where each rank's entry pointer (N + r) ends: follow the earlier shards' last events back until
// a root, a cycle, or the rank's job-wide first event (a root). Job-wide event ids are rank-major over
// the whole job (the unsharded numbering): id = job offset of the rank + its events on earlier shards +
// the local offset.
scan_status blame_shard_tables(Ctx& c, uint64_t N) {
  const uint32_t W = (uint32_t)c.W, G = (uint32_t)c.n_shards, g = (uint32_t)c.shard;
  const size_t row = 5 * (size_t)W;
  CK(c.bl_xs.ensure(row * 4)); CK(c.bl_xr.ensure((size_t)G * row * 4));
  CK(c.bl_gbase.ensure((size_t)W * 8)); CK(c.bl_ext.ensure((size_t)W * 16));
  k_bl_ltab<<<nbk(W, 256), 256, 0, c.stream>>>(W, N, c.rank_off.as<uint64_t>(), c.bl_pa.as<uint32_t>(), c.bl_rk.as<uint16_t>(),
                                                c.bl_xs.as<uint32_t>());
  const int xr = xch_allgather(c, c.bl_xs.p, c.bl_xr.p, row);
  if (xr) { c.err = std::string("blame exchange: ") + xch_error(xr); return SCAN_E_NCCL; }
  std::vector<uint32_t> h((size_t)G * row);
  CK(cudaMemcpyAsync(h.data(), c.bl_xr.p, h.size() * 4, cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  auto L = [&](uint32_t s, uint32_t r, int f) { return h[(size_t)s * row + 4 * (size_t)r + f]; };
  auto cnt = [&](uint32_t s, uint32_t r) { return (uint64_t)h[(size_t)s * row + 4 * (size_t)W + r]; };
  std::vector<uint64_t> jro(W + 1, 0), pre((size_t)G * W, 0);
  for (uint32_t r = 0; r < W; ++r) {
    uint64_t t = 0;
    for (uint32_t s = 0; s < G; ++s) { pre[(size_t)s * W + r] = t; t += cnt(s, r); }
    jro[r + 1] = jro[r] + t;
  }
  auto gid = [&](uint32_t s, uint32_t r, uint64_t k) { return jro[r] + pre[(size_t)s * W + r] + k; };
  std::vector<uint64_t> gb(W);
  std::vector<uint32_t> ext((size_t)W * 4, 0);
  for (uint32_t r = 0; r < W; ++r) {
    gb[r] = gid(g, r, 0) - c.h_rank_off[r];  // + local event index (wraps, then adds back)
    uint32_t rr = r, from = g;
    int64_t s = (int64_t)g - 1;
    uint64_t root = 0;
    uint32_t rrk = 0, ok = 1;
    for (;;) {
      if (s < 0) { root = gid(from, rr, 0); rrk = rr; break; }  // the rank's job-wide first event: a root
      if (cnt((uint32_t)s, rr) == 0) { --s; continue; }       // no events of the rank on shard s
      const uint32_t t = L((uint32_t)s, rr, 0);
      if (t == 0) { rrk = L((uint32_t)s, rr, 1); root = gid((uint32_t)s, rrk, L((uint32_t)s, rr, 2)); break; }
      if (t == 2) { ok = 0; break; }
      from = (uint32_t)s; rr = L((uint32_t)s, rr, 1); --s;  // shard s's first event of rank rr: go on before it
    }
    ext[4 * (size_t)r] = (uint32_t)root; ext[4 * (size_t)r + 1] = (uint32_t)(root >> 32);
    ext[4 * (size_t)r + 2] = rrk; ext[4 * (size_t)r + 3] = ok;
  }
  CK(cudaMemcpyAsync(c.bl_gbase.p, gb.data(), (size_t)W * 8, cudaMemcpyHostToDevice, c.stream));
  CK(cudaMemcpyAsync(c.bl_ext.p, ext.data(), (size_t)W * 16, cudaMemcpyHostToDevice, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  return SCAN_OK;
}

}  // namespace

scan_status blame_all(Ctx& c, scan_blame_result* out) {
  const uint64_t N = c.N, W = c.W;
  const bool sharded = c.n_shards > 1;
  if (N + W >= 0xFFFFFFF0ull) { c.err = "event-level blame supports < 2^32 - 16 - world events per GPU"; return SCAN_E_UNSUPPORTED; }
  scan_status st = ensure_tiles(c);
  if (st) return st;
  if (c.xwait_pending) {  // comm-order view of the cross-stage waits
    launch_xwait_scatter(c);
    c.xwait_pending = false;
  }
  const uint64_t N1 = std::max<uint64_t>(N, 1);
  // jumping lists (bl_inst, bl_pb): jb block segments of S entries
  const unsigned jb = (unsigned)std::min<uint64_t>(nbk(N, JB_NT), 148ull * 8);
  const uint64_t S = (N + (uint64_t)jb * JB_NT - 1) / ((uint64_t)jb * JB_NT) * JB_NT;  // elements per block in round 1
  const uint64_t LCAP = std::max<uint64_t>(N1, (uint64_t)jb * S);
  CK(c.bl_inst.ensure(LCAP * 4)); CK(c.bl_pa.ensure(N1 * 4));
  CK(c.bl_pb.ensure(LCAP * 4)); CK(c.bl_root.ensure(N1 * 8)); CK(c.bl_rk.ensure(N1 * 2)); CK(c.bl_last.ensure(std::max<uint64_t>(c.n_inst, 1) * 4));
  CK(c.bl_rank.ensure(4 * W * 8 + 16 + 8));
  flush_fills(c);
  CK(cudaMemsetAsync(c.bl_rank.p, 0, 4 * W * 8 + 16 + 8, c.stream));
  int launches = 0;
  // the blame kernels read the comm-order instance ids and waits directly (no event-order expansion)
  unsigned int* counters2 = reinterpret_cast<unsigned int*>(c.bl_rank.as<uint8_t>() + 4 * W * 8 + 16);  // [0] changed, [1] n_active
  BA b{c.n_tiles, c.tile_rank.as<uint32_t>(), c.tile_start.as<uint64_t>(), c.rank_off.as<uint64_t>(), c.d_kind,
       c.inst_c.as<uint32_t>(), c.wait_c.as<uint32_t>(), c.inst_rec.as<uint4>(), c.r_comm_off.as<uint64_t>(),
       c.t_commpre.as<uint32_t>(), c.bl_last.as<uint32_t>(), nullptr, c.bl_rk.as<uint16_t>(), c.bl_pa.as<uint32_t>(),
       counters2 + 1, (sharded && c.shard > 0) ? 1u : 0u, N, tile_order_ptr(c)};
  const unsigned tb = nbk(c.n_tiles, 8);
  uint32_t rounds = 0;
  unsigned int n_act = 0;
  unsigned int* changed = counters2;
  const uint32_t* src = c.bl_pa.as<uint32_t>();
  if (N) {
    launches += timed(c, "k_bl_ptr", [&] {
      k_bl_last<<<tb, 256, 0, c.stream>>>(b);
      k_bl_ptr<<<tb, 256, 0, c.stream>>>(b);
      return 2;
    });
    CK(cudaMemcpyAsync(&n_act, counters2 + 1, 4, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    // pointer jumping until no pointer changes (2^34 > N steps at most): round 1 over every event,
    // later rounds over the per-block lists of events whose pointer moved (list buffers bl_inst, bl_pb)
    CK(c.bl_seg.ensure(2ull * jb * 4));
    uint32_t* lists[2] = {c.bl_inst.as<uint32_t>(), c.bl_pb.as<uint32_t>()};
    uint32_t* segs[2] = {c.bl_seg.as<uint32_t>(), c.bl_seg.as<uint32_t>() + jb};
    int cur = 0;
    while (n_act && rounds < 34) {
      CK(cudaMemsetAsync(changed, 0, 4, c.stream));
      launches += timed(c, "k_bl_jump", [&] {
        if (rounds == 0) k_bl_jump0<<<jb, JB_NT, 0, c.stream>>>(N, S, c.bl_pa.as<uint32_t>(), lists[0], segs[0], changed);
        else k_bl_jumpk<<<jb, JB_NT, 0, c.stream>>>(N, S, c.bl_pa.as<uint32_t>(), lists[cur], segs[cur], lists[cur ^ 1],
                                                    segs[cur ^ 1], changed);
        return 1;
      });
      if (rounds > 0) cur ^= 1;
      ++rounds;
      unsigned int h = 0;
      CK(cudaMemcpyAsync(&h, changed, 4, cudaMemcpyDeviceToHost, c.stream));
      CK(cudaStreamSynchronize(c.stream));
      if (!h) break;
    }
    unsigned long long* R = c.bl_rank.as<unsigned long long>();
    const bool sh = W * 8 <= 96 * 1024;
    SA sa{b, (uint32_t)W, src, c.bl_root.as<unsigned long long>(), R, R + W, R + 2 * W, R + 3 * W, R + 4 * W, sh ? 1 : 0,
          nullptr, nullptr};
    if (sharded) {  // the chains that leave the shard: resolved over the earlier shards' per-rank tables
      if ((st = blame_shard_tables(c, N))) return st;
      sa.gbase = c.bl_gbase.as<unsigned long long>(); sa.ext = c.bl_ext.as<uint4>();
      launches += 1;
    }
    const size_t smem = sh ? W * 8 : 0;
    if (smem > 48 * 1024) CK(cudaFuncSetAttribute(k_bl_sum, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned sb = (unsigned)std::min<uint64_t>(tb, 148ull * MS_BS_MINB);
    launches += timed(c, "k_bl_sum", [&] { k_bl_sum<<<sb, 256, smem, c.stream>>>(sa); return 1; });
  } else if (sharded) {  // no local events: still take part in the exchange
    if ((st = blame_shard_tables(c, 0))) return st;
  }
  if (sharded) {  // job-wide per-rank sums and counters
    xch_group_start(c);
    xch_allreduce(c, c.bl_rank.p, 4 * W + 2, XU64);
    const int xr = xch_group_end(c);
    if (xr) { c.err = std::string("blame all-reduce: ") + xch_error(xr); return SCAN_E_NCCL; }
  }
  c.launches += launches;
  std::vector<unsigned long long> h(4 * W + 2);
  CK(cudaMemcpyAsync(h.data(), c.bl_rank.p, (4 * W + 2) * 8, cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  CK(cudaGetLastError());
  if (out) {
    *out = scan_blame_result{};
    out->n_waiting = h[4 * W]; out->n_cyclic = h[4 * W + 1]; out->rounds = rounds; out->top_rank = 0xFFFFFFFFu;
    out->n_active = n_act;
    unsigned long long best = 0;
    for (uint64_t r = 0; r < W; ++r) {
      out->total_wait_ns += h[3 * W + r];
      if (h[r] > best) { best = h[r]; out->top_rank = (uint32_t)r; }
    }
  }
  c.blamed = true;
  return SCAN_OK;
}

}  // namespace ms

using namespace ms;

extern "C" scan_status scan_blame(scan_ctx* ctx, scan_blame_result* out) {
  if (!ctx) return SCAN_E_INVALID_ARG;
  Ctx& c = ctx->c;
  CK(cudaSetDevice(c.device));
  // sharded contexts: a collective call (every shard), job-wide per-rank sums and event ids
  if (c.stream_mode) { c.err = "event-level blame is unavailable on stream contexts"; return SCAN_E_UNSUPPORTED; }
  if (!c.localized) { c.err = "scan_blame needs a completed analysis (scan_analyze or scan_localize)"; return SCAN_E_ORDER; }
  return blame_all(c, out);
}
