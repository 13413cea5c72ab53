// k_stage.cu — K9 v2: the persistent, TMA-fed fused SPMD stage pass (the hot path of scan_analyze).
//
// Same method and outputs as k_fused_t (k_fused.cu), re-laid out for sm_100a. Inside one pipeline
// stage every TP x DP rank runs the same op sequence ("identical sequences of compute
// kernels"), so position p of the stage's template is the same logical op on every rank row:
//   * compute position: stage 1 over the DP peers of every TP index;
//   * TP / DP collective position: the TP / DP group instances -- matching, the
//     decomposition, stage 2 and the wait-for edges;
//   * cross-stage position (P2P, model-parallel, embedding): member slots for k_cross_reduce.
//
// One CTA per SM owns a contiguous range of the job's stage tiles (T positions x R = TP*DP rank rows)
// and walks it in order:
//   * a producer warp streams each tile's rank rows of dur / comm / kind_op and the template words
//     into a 2-stage shared-memory ring with cp.async.bulk (TMA) copies completing on mbarriers, so
//     the DRAM stream of tile i+1 overlaps the compute of tile i;
//   * 15 consumer warps run phase A (micro-tiles of 4 positions x all rows, one 16-byte shared load
//     per row: kind verification, stage 1 with an exact quick reject, per-rank compute sums), then
//     phase B (the tile's communication positions round-robin over the warps: comm verification,
//     group min / max / last arriver by warp shuffles, waits, instance records, stage 2, edges), then
//     a coalesced flush of the per-rank instance ids and waits staged in place in the tile buffer;
//   * per-rank sums and stage-1 / stage-2 counters live in registers for the whole range, wait-for
//     edge weights in shared memory; all are flushed once per range / window / stage.
// Stage 2's "preceding computation" (pslow: any stage-1-slow compute op since the rank's previous
// communication event) is carried from tile to tile in a per-row flag; at the start of a range the
// CTA recomputes the stage-1 bits of the compute positions between the previous communication
// position and its first tile, so no tile-boundary deferral pass exists. P2P payload / warm-up
// gathers are left to k_cross_reduce (this kernel stores the member's position), so no dependent
// global load sits between two barriers. Any verification failure sets NOT_SPMD and the analysis
// reruns the general path (api.cu).
#include "internal.cuh"

#include <cuda.h>

#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <cstring>
#include <cstdio>

namespace ms {

constexpr int SG_NCW = 15;                // consumer warps (+1 producer = 16 warps: 128 registers per thread)
constexpr int SG_NT = 32 * (SG_NCW + 1);  // + one producer warp (TMA issue)
constexpr int SG_NS = 2;                  // ring stages
constexpr uint32_t SG_NPR = 4;            // P2P roles per stage with a cached channel table
constexpr uint32_t SG_TBW = 40;           // words of the tile-major record (k_fused_scan)

namespace {

enum : uint32_t { SG_COMPUTE = 0, SG_TP = 1, SG_DP = 2, SG_XCOLL = 3, SG_P2P = 4 };
constexpr uint32_t SG_BAR_A = 1, SG_BAR_B = 2, SG_BAR_C = 3;  // named barriers of the consumer warps

// ----------------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @p bra DONE_%=;\n bra WAIT_%=;\n"
      "DONE_%=:\n}" ::"r"(bar), "r"(parity) : "memory");
}
// bulk copy global -> shared on the TMA engine; completion counted in bytes on an mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
// 2-D tensor copy (TMA, 128-byte swizzle) of box {x .. x+bx, y .. y+by} of the map at tmap (global memory)
__device__ __forceinline__ void tma_2d(uint32_t dst, const void* tmap, int x, int y, uint32_t bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(dst), "l"(tmap), "r"(x), "r"(y), "r"(bar) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bar_sync(uint32_t id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(32 * SG_NCW) : "memory");
}

}  // namespace

struct StageArgs {
  const uint32_t* dur; const uint16_t* kind; const uint32_t* comm;
  uint64_t n_events;
  const uint64_t* rank_off;
  int TP, DP, PP, W; uint32_t n_comms;
  uint32_t T, R, n_ftiles, n_cta;
  const uint32_t* st_tile0; const uint32_t* st_npos; const uint32_t* st_tot;
  const uint32_t* posA; const uint32_t* posB; const uint16_t* posK;
  const uint32_t* tbase;       // [tile][SG_TBW]: FCOLS scanned bases, comm count, compute count, stage
  const uint32_t* role_comm; const uint32_t* role_slot; const uint32_t* ncroles; const uint8_t* role_type; uint32_t NCRM;
  const uint32_t* eidx; const uint64_t* coff;
  const uint64_t* ch_base; const uint64_t* ch_slot; const uint32_t* bitmap; const uint32_t* bitpre;
  const uint64_t* comm_off; const uint64_t* comp_off; const uint64_t* bits_off;
  uint32_t* inst_c; uint32_t* wait_c; uint32_t* bits; uint32_t* cref; uint4* rec;
  uint4* slots;  // SlotRec per member slot (P2P: w = the event's position in its rank, k_cross_reduce gathers)
  uint64_t p2p_slot0, p2p_inst0;
  uint32_t* citer; uint32_t NIT1;
  uint64_t nnz_tot;
  unsigned long long* ew; unsigned long long* rk_sum; uint32_t* wl_joined; uint32_t* wl_late;
  uint32_t* wd_total; uint32_t* wd_slow;
  uint32_t slow_num, slow_den; unsigned long long slow_margin;
  uint32_t wi, classes, mode; unsigned long long late_margin, wait_margin; int want_ref;
  unsigned long long wi_m;
  uint32_t it_off;
  Counters* cnt;
  unsigned long long* dbg;  // exp & 64: per-CTA phase cycle counts [n_cta][8] (warp 0)
  uint32_t exp;  // timing experiments only (MS_STAGE_EXP, results invalid when set): 1 skip the full stage 1, 2 skip slow-bit
                 // atomics, 4 skip stage-2 counting
  // TMA tensor maps [PP][3] (dur, comm, kind) in global memory, 64-byte aligned (CUtensorMap, 128 B each):
  // per stage block a 2-D view {npos (positions), R (rank rows)}, 128-byte swizzle, boxes of 128 bytes x R
  const uint8_t* tmaps; int kind2d;  // kind2d = 0: kind rows by per-row 1-D bulk copies (rows not 16-byte aligned)
  // shared-memory layout (host-computed, stage_layout)
  uint32_t RGN, KRGN, RSK, SWD, ES, NRT;  // dur / comm region bytes per 32 positions, kind region bytes per 64 positions,
                                          // kind row stride (1-D fallback, bytes), slow-bit words / row, edge row
                                          // stride, role-table entries per row
  uint32_t stage_bytes, o_dur, o_comm, o_kind, o_pa, o_pb, o_pk, o_tb, o_sb, o_cpos, o_ctl;  // within a stage
  uint32_t o_bar, o_edge, o_coffr, o_rt, o_rmap, o_cflag, o_glob, o_st, o_strb, o_slowc, o_boff, o_rel;
};

namespace {

// F(integral_constant<int, 0>) ... F(integral_constant<int, N-1>): compile-time indices into register arrays
template <int I, int N, class F>
__device__ __forceinline__ void static_for_i(F&& f) {
  if constexpr (I < N) { f(std::integral_constant<int, I>{}); static_for_i<I + 1, N>(f); }
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) { static_for_i<0, N>(f); }

__device__ __forceinline__ uint32_t sg_win(const StageArgs& a, uint32_t it) {
  return a.wi == 0 ? 0u : (a.wi == 1 ? it : (uint32_t)__umul64hi((unsigned long long)it, a.wi_m));
}

// word offset of (row, position p) in a dur / comm tile: one 128-byte-swizzled TMA region per 32
// positions ([R][128 B], the 16-byte chunk c of row r stored at chunk c ^ (r & 7)), so 16-byte loads of
// 4 positions by 8 consecutive rows hit 8 distinct bank groups
__device__ __forceinline__ uint32_t dc(const StageArgs& a, uint32_t row, uint32_t p) {
  return (p >> 5) * (a.RGN >> 2) + row * 32u + ((((p >> 2) & 7u) ^ (row & 7u)) << 2) + (p & 3u);
}
// byte offset of (row, p) in the kind tile: swizzled TMA regions of 64 positions, or (1-D fallback)
// per-row 16-byte covers with the row's start shift ksh
__device__ __forceinline__ uint32_t kc(const StageArgs& a, uint32_t row, uint32_t p, uint32_t ksh) {
  return a.kind2d ? (p >> 6) * a.KRGN + row * 128u + ((((p >> 3) & 7u) ^ (row & 7u)) << 4) + ((p & 7u) << 1)
                  : row * a.RSK + ksh + 2 * p;
}

// any slow bit of a row's tile bits over positions [lo, hi)
__device__ __forceinline__ bool seg_any(const uint32_t* b, uint32_t lo, uint32_t hi) {
  if (lo >= hi) return false;
  const uint32_t w0 = lo >> 5, w1 = (hi - 1) >> 5;
  for (uint32_t w = w0; w <= w1; ++w) {
    uint32_t m = b[w];
    if (w == w0) m &= 0xFFFFFFFFu << (lo & 31);
    if (w == w1) m &= 0xFFFFFFFFu >> (31 - ((hi - 1) & 31));
    if (m) return true;
  }
  return false;
}

// Stage 1 at one compute position (readings R8, R15): leave-one-out lower median of the
// OTHER DP peers; slow iff den*x > num*ref and x > ref + margin. x[k] = this lane's row l + 32k. The
// DP group of lane l is every row with the same TP index (l mod TP). Its min / max decide exactly
// whether anyone can be slow (ref >= group min): den*max <= num*min -> nobody. Only then (or when
// references are exported) the full network runs: every lane sorts its group's DP values
// (fetch(d) = value of DP index d), padded to P with sentinels so the two middle order statistics
// land at P/2-1, P/2, and ref = x > va ? va : vb. Returns the slow bits of the lane's rows.
template <int NRB, int P, class Fetch>
__device__ __forceinline__ uint32_t sg_stage1(const StageArgs& a, const uint32_t (&x)[NRB], uint32_t vmask, uint32_t TP,
                                              uint32_t DP, Fetch fetch, uint32_t (&ref)[NRB], bool& full) {
  uint32_t mn = 0xFFFFFFFFu, mx = 0;
#pragma unroll
  for (int k = 0; k < NRB; ++k)
    if ((vmask >> k) & 1u) { mn = min(mn, x[k]); mx = max(mx, x[k]); }
  for (uint32_t m = TP; m < 32; m <<= 1) {
    mn = min(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, m));
    mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, m));
  }
  const bool maybe = vmask && (unsigned long long)a.slow_den * mx > (unsigned long long)a.slow_num * mn;
  uint32_t slow = 0;
  full = __any_sync(0xFFFFFFFFu, maybe) || a.want_ref;
  if (full) {  // warp-uniform rare path
    const int q = ((int)DP - 2) / 2;
    const int L = P / 2 - 1 - q;
    uint32_t v[P];
#pragma unroll
    for (int d = 0; d < P; ++d) v[d] = d < (int)DP ? fetch((uint32_t)d) : (d < (int)DP + L ? 0u : 0xFFFFFFFFu);
#pragma unroll
    for (int kk = 2; kk <= P; kk <<= 1)
#pragma unroll
      for (int jj = kk >> 1; jj > 0; jj >>= 1)
#pragma unroll
        for (int i = 0; i < P; ++i) {
          const int ixj = i ^ jj;
          if (ixj > i) {
            const bool up = (i & kk) == 0;
            const uint32_t lo = min(v[i], v[ixj]), hi = max(v[i], v[ixj]);
            v[i] = up ? lo : hi; v[ixj] = up ? hi : lo;
          }
        }
    const uint32_t va = v[P / 2 - 1], vb = v[P / 2];
#pragma unroll
    for (int k = 0; k < NRB; ++k) {
      const uint32_t r_ = x[k] > va ? va : vb;
      ref[k] = r_;
      const unsigned long long du = x[k];
      const bool s = ((vmask >> k) & 1u) && (unsigned long long)a.slow_den * du > (unsigned long long)a.slow_num * r_ &&
                     du > (unsigned long long)r_ + a.slow_margin;
      slow |= s ? (1u << k) : 0u;
    }
  }
  return slow;
}

// per-warp register accumulators of the lane's rows (flushed with global atomics)
template <int NRB>
struct Acc {
  unsigned long long comp[NRB], wait[NRB], tr[NRB];
  uint32_t join[NRB], late[NRB];
  uint32_t tot;           // compute positions of the current stage-1 window (same for every row)
  uint32_t w1, w2;        // windows of the stage-1 / stage-2 counters
};

template <int NRB>
__device__ __forceinline__ void flush_s1(const StageArgs& a, Acc<NRB>& c, uint32_t sbase, uint32_t lane) {
#pragma unroll
  for (int k = 0; k < NRB; ++k) {
    const uint32_t row = lane + 32u * k;
    if (row < a.R) {
      const uint64_t o = (uint64_t)c.w1 * a.W + sbase + row;
      if (c.tot) atomicAdd(&a.wd_total[o], c.tot);
    }
  }
  c.tot = 0;
}

template <int NRB>
__device__ __forceinline__ void flush_s2(const StageArgs& a, Acc<NRB>& c, uint32_t sbase, uint32_t lane) {
#pragma unroll
  for (int k = 0; k < NRB; ++k) {
    const uint32_t row = lane + 32u * k;
    if (row < a.R) {
      const uint64_t o = (uint64_t)c.w2 * a.W + sbase + row;
      if (c.join[k]) atomicAdd(&a.wl_joined[o], c.join[k]);
      if (c.late[k]) atomicAdd(&a.wl_late[o], c.late[k]);
    }
    c.join[k] = 0; c.late[k] = 0;
  }
}

template <int NRB>
__device__ __forceinline__ void flush_sums(const StageArgs& a, Acc<NRB>& c, uint32_t sbase, uint32_t lane) {
#pragma unroll
  for (int k = 0; k < NRB; ++k) {
    const uint32_t row = lane + 32u * k;
    if (row < a.R) {
      const uint32_t r = sbase + row;
      if (c.comp[k]) atomicAdd(&a.rk_sum[r], c.comp[k]);
      if (c.wait[k]) atomicAdd(&a.rk_sum[a.W + r], c.wait[k]);
      if (c.tr[k]) atomicAdd(&a.rk_sum[2 * a.W + r], c.tr[k]);
    }
    c.comp[k] = 0; c.wait[k] = 0; c.tr[k] = 0;
  }
}

// the shared-memory wait-for edge sums and stage-1 slow counts of the current (window, stage) -> global, then zero
__device__ __forceinline__ void flush_edges(const StageArgs& a, uint32_t* edge, uint32_t* slowc, uint32_t sbase, uint32_t win,
                                            uint32_t ctid) {
  for (uint32_t r = ctid; r < a.R; r += 32 * SG_NCW) {
    const uint32_t v = slowc[r];
    if (v) { slowc[r] = 0; atomicAdd(&a.wd_slow[(uint64_t)win * a.W + sbase + r], v); }
  }
  const uint32_t E = (uint32_t)(a.TP + a.DP);
  for (uint32_t i = ctid; i < a.R * a.ES; i += 32 * SG_NCW) {
    const uint32_t v = edge[i];
    if (!v) continue;
    edge[i] = 0;
    const uint32_t row = i / a.ES, slot = i - row * a.ES;
    atomicAdd(&a.ew[(uint64_t)win * a.nnz_tot + a.eidx[(uint64_t)(sbase + row) * E + slot]], (unsigned long long)v);
  }
}

}  // namespace

template <int NRB, int P>
__global__ void __launch_bounds__(SG_NT, 1) k_stage(const __grid_constant__ StageArgs a) {
  extern __shared__ __align__(128) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);  // swizzled TMA destinations: 1024-aligned
  const uint32_t tid = threadIdx.x, wid = tid >> 5, lane = lane_id();
  const uint32_t T = a.T, R = a.R, TP = (uint32_t)a.TP, DP = (uint32_t)a.DP;
  const uint32_t tpsh = __ffs(TP) - 1;
  const uint32_t t_begin = (uint32_t)((uint64_t)blockIdx.x * a.n_ftiles / a.n_cta);
  const uint32_t t_end = (uint32_t)((uint64_t)(blockIdx.x + 1) * a.n_ftiles / a.n_cta);
  const uint32_t bar0 = smem_u32(sm + a.o_bar);  // full[s] at bar0 + 8s, empty[s] at bar0 + 8(NS + s)
  uint32_t* st_tab = reinterpret_cast<uint32_t*>(sm + a.o_st);  // [PP+1] st_tile0, then [PP] st_npos
  uint64_t* st_rb = reinterpret_cast<uint64_t*>(sm + a.o_strb);   // [PP] first event of each stage block
  if (tid == 0) {
    for (int s = 0; s < SG_NS; ++s) { mbar_init(bar0 + 8 * s, 32); mbar_init(bar0 + 8 * (SG_NS + s), SG_NCW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int s = 0; s < SG_NS; ++s) {  // per-stage slow bits and flags start clear (then kept clear after each use)
    uint32_t* sbz = reinterpret_cast<uint32_t*>(sm + (uint64_t)s * a.stage_bytes + a.o_sb);
    for (uint32_t i = tid; i < R * a.SWD; i += SG_NT) sbz[i] = 0;
    if (tid == 0) reinterpret_cast<uint32_t*>(sm + (uint64_t)s * a.stage_bytes + a.o_ctl)[0] = 0;
  }
  for (uint32_t i = tid; i <= (uint32_t)a.PP; i += SG_NT) st_tab[i] = a.st_tile0[i];
  for (uint32_t i = tid; i < (uint32_t)a.PP; i += SG_NT) { st_tab[a.PP + 1 + i] = a.st_npos[i]; st_rb[i] = a.rank_off[(uint64_t)i * R]; }
  __syncthreads();
  if (t_begin >= t_end) return;
  auto stage_of = [&](uint32_t t) {
    uint32_t st = 0;
    while (st + 1 < (uint32_t)a.PP && st_tab[st + 1] <= t) ++st;
    return st;
  };

  // ---- TMA issue of tile t into ring slot s by one whole warp (32 arrivals on full[s] + the tx bytes)
  auto issue = [&](uint32_t t, uint32_t s) {
    const uint32_t st = stage_of(t);
    const uint32_t npos = st_tab[a.PP + 1 + st];
    const uint32_t p0 = (t - st_tab[st]) * T, np = min(T, npos - p0);
    const uint64_t rbase = st_rb[st];
    uint8_t* sb = sm + (uint64_t)s * a.stage_bytes;
    const uint32_t bar = bar0 + 8 * s;
    // tx bytes: template words, dur / comm boxes (R x 128 B per 32 positions, full boxes even past the
    // stage's end: TMA zero-fills out-of-bound elements), kind boxes or per-row 16-byte covers
    const uint32_t H = (np + 31) / 32, HK = (np + 63) / 64;
    uint32_t kb = 0;
    if (!a.kind2d) {
      for (uint32_t row = lane; row < R; row += 32) {
        const uint64_t e0 = rbase + (uint64_t)row * npos + p0;
        const uint64_t b0 = (2 * e0) & ~15ull, b1 = (2 * (e0 + np) + 15) & ~15ull;
        if (b1 <= 2 * a.n_events) kb += (uint32_t)(b1 - b0);
      }
      for (int o = 16; o > 0; o >>= 1) kb += __shfl_xor_sync(0xFFFFFFFFu, kb, o);
    } else {
      kb = HK * R * 128;
    }
    const uint32_t ta = (np * 4 + 15) & ~15u, tk = (np * 2 + 15) & ~15u;
    if (lane == 0) mbar_expect_tx(bar, 2 * ta + tk + SG_TBW * 4 + 2 * H * R * 128 + kb);
    __syncwarp();
    const uint8_t* maps = a.tmaps + (uint64_t)st * 3 * 128;
    if (lane == 0) {
      bulk_g2s(smem_u32(sb + a.o_pa), a.posA + (uint64_t)t * T, ta, bar);
      bulk_g2s(smem_u32(sb + a.o_pb), a.posB + (uint64_t)t * T, ta, bar);
      bulk_g2s(smem_u32(sb + a.o_pk), a.posK + (uint64_t)t * T, tk, bar);
      bulk_g2s(smem_u32(sb + a.o_tb), a.tbase + (uint64_t)t * SG_TBW, SG_TBW * 4, bar);
    }
    for (uint32_t h = lane; h < H; h += 32) {
      tma_2d(smem_u32(sb + a.o_dur + h * a.RGN), maps, (int)(p0 + 32 * h), 0, bar);
      tma_2d(smem_u32(sb + a.o_comm + h * a.RGN), maps + 128, (int)(p0 + 32 * h), 0, bar);
    }
    if (a.kind2d) {
      for (uint32_t h = lane; h < HK; h += 32) tma_2d(smem_u32(sb + a.o_kind + h * a.KRGN), maps + 256, (int)(p0 + 64 * h), 0, bar);
    } else {
      for (uint32_t row = lane; row < R; row += 32) {
        const uint64_t e0 = rbase + (uint64_t)row * npos + p0;
        const uint64_t b0 = (2 * e0) & ~15ull, b1 = (2 * (e0 + np) + 15) & ~15ull;
        uint8_t* kd = sb + a.o_kind + row * a.RSK;
        if (b1 <= 2 * a.n_events) {
          bulk_g2s(smem_u32(kd), reinterpret_cast<const uint8_t*>(a.kind) + b0, (uint32_t)(b1 - b0), bar);
        } else {  // the column's last row: the 16-byte cover would run past the column, copy by elements
          const uint32_t sh = (uint32_t)((2 * e0) & 15ull) / 2;
          for (uint32_t q = 0; q < np; ++q) reinterpret_cast<uint16_t*>(kd)[sh + q] = a.kind[e0 + q];
        }
      }
    }
    mbar_arrive(bar);
  };
  // =========================================================================== producer warp
  if (wid == SG_NCW) {
    for (uint32_t t = t_begin, i = 0; t < t_end; ++t, ++i) {
      const uint32_t s = i % SG_NS, use = i / SG_NS;
      if (use) mbar_wait(bar0 + 8 * (SG_NS + s), (use - 1) & 1u);  // the consumers released this slot
      issue(t, s);
    }
    return;
  }

  // =========================================================================== consumer warps
  const uint32_t ctid = tid;  // 0 .. 32*NCW-1
  uint32_t* edge = reinterpret_cast<uint32_t*>(sm + a.o_edge);          // [R][ES] current (window, stage)
  unsigned long long* coffr = reinterpret_cast<unsigned long long*>(sm + a.o_coffr);  // [R] comm offsets
  // role table, role-major so a warp's lanes (consecutive rows) read consecutive words: [NRT][R] {expected
  // comm / peer, channel base}, then [NRT][R] {slot base, member count | slot << 16 | send << 31}
  uint2* rtx = reinterpret_cast<uint2*>(sm + a.o_rt);
  uint2* rtz = rtx + (size_t)a.NRT * R;
  uint8_t* rmap = sm + a.o_rmap;                                        // [ROLES] role -> table entry (0xFF none)
  uint32_t* cflag = reinterpret_cast<uint32_t*>(sm + a.o_cflag);        // [R] pslow carried into the next tile
  uint32_t* glob = reinterpret_cast<uint32_t*>(sm + a.o_glob);          // [0] any cflag
  uint32_t* slowc = reinterpret_cast<uint32_t*>(sm + a.o_slowc);        // [R] stage-1 slow events of the current window
  unsigned long long* boff = reinterpret_cast<unsigned long long*>(sm + a.o_boff);  // [R] first slow-bit word of each row
  for (uint32_t i = ctid; i < R; i += 32 * SG_NCW) slowc[i] = 0;
  for (uint32_t i = ctid; i < R * a.ES; i += 32 * SG_NCW) edge[i] = 0;
  for (uint32_t i = ctid; i < R; i += 32 * SG_NCW) cflag[i] = 0;
  if (ctid == 0) glob[0] = 0;

  Acc<NRB> acc;
#pragma unroll
  for (int k = 0; k < NRB; ++k) { acc.comp[k] = acc.wait[k] = acc.tr[k] = 0; acc.join[k] = acc.late[k] = 0; }
  acc.tot = 0; acc.w1 = 0; acc.w2 = 0;
  uint32_t vmask = 0;
#pragma unroll
  for (int k = 0; k < NRB; ++k) vmask |= (lane + 32u * k < R) ? (1u << k) : 0u;

  // ---- stage-2 carry at the start of the range (mode 0): the stage-1 bits of the compute positions
  // between the previous communication position and the first tile (owned by the previous range)
  bar_sync(SG_BAR_C);
  if (a.mode == 0 && DP >= 2) {
    const uint32_t st = stage_of(t_begin);
    if (t_begin > st_tab[st]) {
      const uint32_t* tb = a.tbase + (uint64_t)t_begin * SG_TBW;
      const uint32_t j0 = tb[ROLES], jp0 = tb[ROLES + 3];
      const uint32_t npos = st_tab[a.PP + 1 + st], p0 = (t_begin - st_tab[st]) * T;
      const uint64_t rbase = st_rb[st];
      const uint32_t L = j0 - jp0;  // compute positions right before p0 (no comm position between)
      bool any = false;
      for (uint32_t i = wid; i < L; i += SG_NCW) {
        const uint32_t pos = p0 - L + i;
        uint32_t x[NRB], ref[NRB];
#pragma unroll
        for (int k = 0; k < NRB; ++k) x[k] = ((vmask >> k) & 1u) ? a.dur[rbase + (uint64_t)(lane + 32u * k) * npos + pos] : 0u;
        const uint32_t tp = lane & (TP - 1);
        bool full;
        const uint32_t sl = sg_stage1<NRB, P>(a, x, vmask, TP, DP,
                                              [&](uint32_t d) { return a.dur[rbase + (uint64_t)(tp + TP * d) * npos + pos]; }, ref, full);
#pragma unroll
        for (int k = 0; k < NRB; ++k)
          if ((sl >> k) & 1u) { atomicOr(&cflag[lane + 32u * k], 1u); any = true; }
      }
      if (__any_sync(0xFFFFFFFFu, any) && lane == 0) glob[0] = 1;
    }
  }

  // per-lane constants of the swizzled tiles: this lane's rows are lane + 32k, so row & 7 == lane & 7
  const uint32_t rx = (lane & 7u) << 2, kx = (lane & 7u) << 3, lb = lane * 32u, lbk = lane * 64u;
  const uint32_t RG4 = a.RGN >> 2, KR2 = a.KRGN >> 1;
  auto pw = [&](uint32_t p) { return (p >> 5) * RG4 + (p & 31u); };   // position part of a dur / comm word offset
  auto kw = [&](uint32_t p) { return (p >> 6) * KR2 + (p & 63u); };   // position part of a kind element offset
  const uint32_t tp = lane & (TP - 1u);
  // ballot mask of the lane's TP group (TP consecutive lanes)
  const uint32_t gmt = TP >= 32 ? 0xFFFFFFFFu : (((1u << TP) - 1u) << (lane & ~(TP - 1u)));

  uint32_t cur_st = 0xFFFFFFFFu, sbase = 0, npos = 0, w_edge = 0;
  uint64_t rbase = 0;
  bool mis = false;
  uint32_t st = stage_of(t_begin);
  unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tk0 = 0, tk1 = 0;
  const bool prof = (a.exp & 64u) && wid == 0;
#define SG_T(ix) do { if (prof) { tk1 = clock64(); ph[ix] += tk1 - tk0; tk0 = tk1; } } while (0)
  if (prof) tk0 = clock64();
  for (uint32_t t = t_begin, i = 0; t < t_end; ++t, ++i) {
    const uint32_t s = i % SG_NS;
    const uint32_t so = s * a.stage_bytes;
    uint32_t* dur_s = reinterpret_cast<uint32_t*>(sm + so + a.o_dur);
    uint32_t* comm_s = reinterpret_cast<uint32_t*>(sm + so + a.o_comm);
    const uint16_t* kind_s = reinterpret_cast<const uint16_t*>(sm + so + a.o_kind);
    const uint32_t* pa = reinterpret_cast<const uint32_t*>(sm + so + a.o_pa);
    const uint32_t* pb = reinterpret_cast<const uint32_t*>(sm + so + a.o_pb);
    const uint16_t* pk = reinterpret_cast<const uint16_t*>(sm + so + a.o_pk);
    const uint32_t* tb = reinterpret_cast<const uint32_t*>(sm + so + a.o_tb);
    uint32_t* sbits = reinterpret_cast<uint32_t*>(sm + so + a.o_sb);    // [R][SWD] slow bits of the tile
    uint16_t* cpos = reinterpret_cast<uint16_t*>(sm + so + a.o_cpos);   // [T] comm positions by comm index
    uint32_t* ctl = reinterpret_cast<uint32_t*>(sm + so + a.o_ctl);     // [0] any slow bit in this tile
    while (st + 1 < (uint32_t)a.PP && st_tab[st + 1] <= t) ++st;
    const uint32_t p0 = (t - st_tab[st]) * T;
    if (st != cur_st) {
      // a new stage block: rows are other ranks. Flush, then reload the stage's tables. The barrier
      // orders this after every warp's flush of the previous tile (which reads coffr).
      bar_sync(SG_BAR_C);
      if (cur_st != 0xFFFFFFFFu) {
        flush_edges(a, edge, slowc, sbase, w_edge, ctid);
        flush_sums(a, acc, sbase, lane);
        flush_s1(a, acc, sbase, lane);
        flush_s2(a, acc, sbase, lane);
        for (uint32_t r = ctid; r < R; r += 32 * SG_NCW) cflag[r] = 0;  // a stage's first comm event: no earlier segment
        if (ctid == 0) glob[0] = 0;
      }
      cur_st = st; sbase = st * R; npos = st_tab[a.PP + 1 + st]; rbase = st_rb[st];
      const uint32_t ncr = a.ncroles[st];
      for (uint32_t r = ctid; r < R; r += 32 * SG_NCW) { coffr[r] = a.comm_off[sbase + r]; boff[r] = a.bits_off[sbase + r]; }
      if (ctid < ROLES) {  // role -> table entry: collective roles in order, present P2P roles after them
        uint32_t e = 0xFFu;
        if (ctid < ncr) e = ctid;
        else if (ctid >= 16 && a.st_tot[(uint64_t)st * FCOLS + ctid]) {
          uint32_t idx = 0;
          for (uint32_t q = 16; q < ctid; ++q) idx += a.st_tot[(uint64_t)st * FCOLS + q] ? 1u : 0u;
          if (idx < SG_NPR) e = a.NCRM + idx;
        }
        rmap[ctid] = (uint8_t)e;
      }
      bar_sync(SG_BAR_C);
      for (uint32_t it = ctid; it < R * ROLES; it += 32 * SG_NCW) {
        const uint32_t row = it / ROLES, ro = it - row * ROLES;
        const uint32_t e = rmap[ro];
        if (e == 0xFFu) continue;
        const uint32_t r = sbase + row;
        uint4 v;
        if (ro < 16) {
          const uint32_t cid = a.role_comm[(uint64_t)r * CROLES + ro];
          const uint32_t nm = (uint32_t)(a.coff[cid + 1] - a.coff[cid]);
          v = make_uint4(cid, (uint32_t)a.ch_base[cid], (uint32_t)a.ch_slot[cid], nm | (a.role_slot[(uint64_t)r * CROLES + ro] << 16));
        } else {
          const int ds = (int)(ro & 7u) - 4;
          const bool send = (ro >> 3) & 1u;
          const int peer = (int)r + ds * (int)R;
          uint32_t b = 0, sl = 0;
          if (peer >= 0 && peer < a.W) {
            const uint32_t src = send ? r : (uint32_t)peer, dst = send ? (uint32_t)peer : r;
            const uint32_t xk = src * (uint32_t)a.W + dst;
            const uint64_t ch = a.n_comms + a.bitpre[xk >> 5] + __popc(a.bitmap[xk >> 5] & ((1u << (xk & 31)) - 1u));
            b = (uint32_t)a.ch_base[ch]; sl = (uint32_t)a.ch_slot[ch];
          }
          v = make_uint4((uint32_t)peer, b, sl, 2u | ((send ? 0u : 1u) << 16) | (send ? 0x80000000u : 0u));
        }
        rtx[e * R + row] = make_uint2(v.x, v.y);
        rtz[e * R + row] = make_uint2(v.z, v.w);
      }
      w_edge = 0xFFFFFFFFu;  // set from the tile's first iteration once its template has landed
    }
    SG_T(0);
    mbar_wait(bar0 + 8 * s, (i / SG_NS) & 1u);  // the tile's bytes have landed
    SG_T(1);
    const uint32_t np = min(T, npos - p0);
    const uint32_t j0 = tb[ROLES], m0 = tb[ROLES + 1], it0 = tb[ROLES + 2];
    const uint32_t cT = tb[FCOLS];
    const uint32_t itg0 = it0 + a.it_off;
    const uint32_t wtile = sg_win(a, itg0);
    if (wtile != w_edge) {  // edge sums of another window: flush (no warp writes edges before BAR_A)
      if (w_edge != 0xFFFFFFFFu) flush_edges(a, edge, slowc, sbase, w_edge, ctid);
      w_edge = wtile;
    }
    // kind element offset of (row, p): swizzled 2-D regions, or the 1-D per-row covers (start shift)
    uint32_t ksh[NRB];
    if (!a.kind2d) {
#pragma unroll
      for (int k = 0; k < NRB; ++k) ksh[k] = (uint32_t)((rbase + (uint64_t)(lane + 32u * k) * npos + p0) & 7ull);
    }

    // ------------------------------------------------------------------ phase A (micro-tiles)
    bool tslow = false;
    const uint32_t nmt = np >> 2;
    for (uint32_t mt = wid; mt < nmt; mt += SG_NCW) {
      const uint32_t pbase = mt * 4;
      const uint2 tk = *reinterpret_cast<const uint2*>(pk + pbase);
      const uint4 A4 = *reinterpret_cast<const uint4*>(pa + pbase);
      const uint4 B4 = *reinterpret_cast<const uint4*>(pb + pbase);
      const uint32_t Kq[4] = {tk.x & 0xFFFFu, tk.x >> 16, tk.y & 0xFFFFu, tk.y >> 16};
      const uint32_t Aq[4] = {A4.x, A4.y, A4.z, A4.w}, Bq[4] = {B4.x, B4.y, B4.z, B4.w};
      // kind_op of every row against the template (P:L144 identical sequences; else NOT_SPMD)
      const uint32_t kq = kw(pbase) ^ kx;
#pragma unroll
      for (int k = 0; k < NRB; ++k)
        if ((vmask >> k) & 1u) {
          const uint32_t ko = a.kind2d ? kq + lbk + 2048u * k : (lane + 32u * k) * (a.RSK >> 1) + ksh[k] + pbase;
          const uint2 kv = *reinterpret_cast<const uint2*>(kind_s + ko);
          mis |= (kv.x != tk.x) | (kv.y != tk.y);
        }
      uint32_t cmask = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) cmask |= ((Kq[q] & 7u) == 0) ? (1u << q) : 0u;
      if (cmask) {
        uint4 dv[NRB];
        const uint32_t wo = (pw(pbase) ^ rx) + lb;
#pragma unroll
        for (int k = 0; k < NRB; ++k)
          dv[k] = ((vmask >> k) & 1u) ? *reinterpret_cast<const uint4*>(dur_s + wo + 1024u * k) : make_uint4(0, 0, 0, 0);
        uint32_t need = 0;  // positions whose DP groups cannot all be exonerated by the quick reject
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (!((cmask >> q) & 1u)) continue;
          uint32_t mn = 0xFFFFFFFFu, mx = 0;
#pragma unroll
          for (int k = 0; k < NRB; ++k) {
            const uint32_t x = q == 0 ? dv[k].x : (q == 1 ? dv[k].y : (q == 2 ? dv[k].z : dv[k].w));
            acc.comp[k] += x;
            if ((vmask >> k) & 1u) { mn = min(mn, x); mx = max(mx, x); }
          }
          if (DP >= 2) {
            if (a.wi) {
              const uint32_t wq = sg_win(a, itg0 + (Bq[q] & 1023u));
              if (wq != acc.w1) { flush_s1(a, acc, sbase, lane); acc.w1 = wq; }
            }
            ++acc.tot;
            for (uint32_t m = TP; m < 32; m <<= 1) {
              mn = min(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, m));
              mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, m));
            }
            const bool maybe = vmask && (unsigned long long)a.slow_den * mx > (unsigned long long)a.slow_num * mn;
            if (__any_sync(0xFFFFFFFFu, maybe) || a.want_ref) need |= 1u << q;
          }
        }
        if (a.exp & 1u) need = 0;
        if (need) {
          // transposed full stage 1 (rare): lane task (q, g) sorts the DP group g at position pbase + q in
          // registers (the DP values of 4 positions x TP groups sit in distinct banks), then decides every
          // member of the group; the slow decisions are gathered by ballots, one shared-memory update per
          // (row, micro-tile) by lane 0
          uint32_t wmask = 0;  // positions of the micro-tile in the tile's window (their counts go to slowc)
#pragma unroll
          for (int q = 0; q < 4; ++q) wmask |= (sg_win(a, itg0 + (Bq[q] & 1023u)) == w_edge) ? (1u << q) : 0u;
          for (uint32_t tb0 = 0; tb0 < 4 * TP; tb0 += 32) {
            const uint32_t task = tb0 + lane;
            const uint32_t q = task / TP, g = task - q * TP;
            const bool act = task < 4 * TP && ((need >> q) & 1u);
            const uint32_t p = pbase + (q & 3u);
            const uint32_t pwp = pw(p);
            const int qm = ((int)DP - 2) / 2;
            const int L = P / 2 - 1 - qm;
            uint32_t v[P];
#pragma unroll
            for (int d = 0; d < P; ++d) {
              const uint32_t row = g + TP * (uint32_t)d;
              v[d] = (act && d < (int)DP) ? dur_s[(pwp ^ ((row & 7u) << 2)) + row * 32u] : (d < (int)DP + L ? 0u : 0xFFFFFFFFu);
            }
#pragma unroll
            for (int kk = 2; kk <= P; kk <<= 1)
#pragma unroll
              for (int jj = kk >> 1; jj > 0; jj >>= 1)
#pragma unroll
                for (int ii = 0; ii < P; ++ii) {
                  const int ixj = ii ^ jj;
                  if (ixj > ii) {
                    const bool up = (ii & kk) == 0;
                    const uint32_t lo = min(v[ii], v[ixj]), hi = max(v[ii], v[ixj]);
                    v[ii] = up ? lo : hi; v[ixj] = up ? hi : lo;
                  }
                }
            const uint32_t va = v[P / 2 - 1], vb = v[P / 2];
            const uint32_t q3 = q & 3u;  // selects, not an indexed (local-memory) array
            const uint32_t Asel = q3 == 0 ? Aq[0] : (q3 == 1 ? Aq[1] : (q3 == 2 ? Aq[2] : Aq[3]));
            const uint32_t j = j0 + (Asel & 1023u);
#pragma unroll 1
            for (uint32_t d = 0; d < DP; ++d) {
              const uint32_t row = g + TP * d;
              bool sl = false;
              if (act) {
                const uint32_t x = dur_s[(pwp ^ ((row & 7u) << 2)) + row * 32u];
                const uint32_t ref = x > va ? va : vb;
                const unsigned long long du = x;
                if (a.want_ref) a.cref[a.comp_off[sbase + row] + j] = ref;
                sl = !(a.exp & 2u) && (unsigned long long)a.slow_den * du > (unsigned long long)a.slow_num * ref &&
                     du > (unsigned long long)ref + a.slow_margin;
              }
              uint32_t b = __ballot_sync(0xFFFFFFFFu, sl);
              while (b) {  // one group g (one row) at a time: its slow positions of the micro-tile as a nibble
                const uint32_t l0 = (uint32_t)(__ffs(b) - 1), t0 = tb0 + l0;
                const uint32_t g0 = t0 - (t0 / TP) * TP, row0 = g0 + TP * d;
                uint32_t nib = 0;
#pragma unroll
                for (uint32_t q2 = 0; q2 < 4; ++q2) {
                  const int l2 = (int)(q2 * TP + g0) - (int)tb0;
                  if (l2 >= 0 && l2 < 32 && ((b >> l2) & 1u)) { nib |= 1u << q2; b &= ~(1u << l2); }
                }
                if (lane == 0 && !(a.exp & 128u)) {
                  atomicOr(&sbits[row0 * a.SWD + (pbase >> 5)], nib << (pbase & 31u));
                  if (nib & wmask) atomicAdd(&slowc[row0], (uint32_t)__popc(nib & wmask));
                  for (uint32_t m2 = nib & ~wmask; m2; m2 &= m2 - 1) {
                    const uint32_t q2 = (uint32_t)(__ffs(m2) - 1);
                    const uint32_t Bsel = q2 == 0 ? Bq[0] : (q2 == 1 ? Bq[1] : (q2 == 2 ? Bq[2] : Bq[3]));
                    atomicAdd(&a.wd_slow[(uint64_t)sg_win(a, itg0 + (Bsel & 1023u)) * a.W + sbase + row0], 1u);
                  }
                }
                tslow = true;
              }
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t p = pbase + q;
        if (!((cmask >> q) & 1u) && lane == 0) {  // a communication position: its comm index -> position (+ class)
          const uint32_t ty = (Bq[q] >> 25) & 7u;
          const uint32_t cls = ty == SG_TP ? 0u : (ty == SG_DP ? 1u : 2u);
          cpos[(Aq[q] >> 10) & 1023u] = (uint16_t)(p | (cls << 12));
        }
        if (Aq[q] >> 31) {  // iteration end: compute index at which the next iteration starts, every row
          const uint32_t v = j0 + (Aq[q] & 1023u) + ((cmask >> q) & 1u);
          const uint32_t itp = it0 + (Bq[q] & 1023u);
#pragma unroll
          for (int k = 0; k < NRB; ++k)
            if ((vmask >> k) & 1u) a.citer[(uint64_t)(sbase + lane + 32u * k) * a.NIT1 + itp + 1] = v;
        }
      }
    }
    if (__any_sync(0xFFFFFFFFu, tslow) && lane == 0) ctl[0] = 1;
    SG_T(2);
    bar_sync(SG_BAR_A);
    SG_T(3);

    // ------------------------------------------------------------------ phase B (comm positions)
    const bool pany = a.mode == 0 && (ctl[0] != 0 || glob[0] != 0);  // any pslow possible in this tile
    const bool s2 = (a.mode != 0 || pany) && !(a.exp & 4u);            // stage-2 counting in this tile
    const uint32_t E = TP + (uint32_t)a.DP;
    for (uint32_t j = wid; j < cT; j += SG_NCW) {
      const uint32_t cv = cpos[j];
      const uint32_t p = cv & 0xFFFu, cls = cv >> 12;  // 0 TP, 1 DP, 2 cross
      const uint32_t Bp = pb[p];
      const uint32_t role = (Bp >> 20) & 31u;
      const uint32_t kinst = tb[role] + ((Bp >> 10) & 1023u);
      const uint32_t itp = itg0 + (Bp & 1023u);
      const uint32_t win = sg_win(a, itp);
      const uint32_t wo = (pw(p) ^ rx) + lb;
      const uint32_t e = rmap[role];
      uint32_t d[NRB], base[NRB];
      // communicator / peer of every row against the role (else NOT_SPMD)
#pragma unroll
      for (int k = 0; k < NRB; ++k) {
        d[k] = 0; base[k] = 0;
        if (!((vmask >> k) & 1u)) continue;
        const uint32_t row = lane + 32u * k;
        d[k] = dur_s[wo + 1024u * k];
        const uint32_t cm = comm_s[wo + 1024u * k];
        uint32_t want;
        if (e != 0xFFu) { const uint2 v = rtx[e * R + row]; want = v.x; base[k] = v.y; }
        else if (role < 16) { want = a.role_comm[(uint64_t)(sbase + row) * CROLES + role]; base[k] = (uint32_t)a.ch_base[want]; }
        else want = (uint32_t)((int)(sbase + row) + ((int)(role & 7u) - 4) * (int)R);
        mis |= cm != want;
      }
      if (cls == 2) {  // cross-stage member: its slot for k_cross_reduce; the tile keeps the instance id
#pragma unroll
        for (int k = 0; k < NRB; ++k) {
          if (!((vmask >> k) & 1u)) continue;
          const uint32_t row = lane + 32u * k, r = sbase + row;
          uint64_t bch, sch;
          uint32_t nm, slot;
          bool send = false;
          if (e != 0xFFu) {
            const uint2 vx = rtx[e * R + row], vz = rtz[e * R + row];
            const uint4 v = make_uint4(vx.x, vx.y, vz.x, vz.y);
            bch = v.y; sch = v.z; nm = v.w & 0xFFFFu;
            slot = role < 16 ? v.w >> 16 : (v.w >> 16) & 1u; send = role >= 16 && (v.w >> 31);
          } else {  // uncached role (more P2P roles than the table holds): global lookups
            uint64_t ch;
            if (role < 16) {
              const uint32_t cid = a.role_comm[(uint64_t)r * CROLES + role];
              ch = cid; nm = (uint32_t)(a.coff[cid + 1] - a.coff[cid]); slot = a.role_slot[(uint64_t)r * CROLES + role];
            } else {
              const int ds = (int)(role & 7u) - 4;
              send = (role >> 3) & 1u;
              const uint32_t peer = (uint32_t)((int)r + ds * (int)R);
              const uint32_t src = send ? r : peer, dst = send ? peer : r;
              const uint32_t xk = src * (uint32_t)a.W + dst;
              ch = a.n_comms + a.bitpre[xk >> 5] + __popc(a.bitmap[xk >> 5] & ((1u << (xk & 31)) - 1u));
              nm = 2; slot = send ? 0 : 1;
            }
            bch = a.ch_base[ch]; sch = a.ch_slot[ch];
          }
          const uint64_t inst = bch + kinst;
          const uint64_t si = sch + (uint64_t)kinst * nm + slot;
          a.slots[si] = make_uint4(d[k], (uint32_t)(coffr[row] + m0 + j), slot_z(itp, pk[p], 0u), role >= 16 ? p0 + p : 0u);
          comm_s[wo + 1024u * k] = (uint32_t)inst;
        }
        continue;
      }
      const bool istp = cls == 0;
      const uint32_t clsid = istp ? 1u : 2u;
      const bool elig = s2 && ((a.classes >> (clsid - 1)) & 1u);
      const bool trans = istp ? TP > 1 : DP > 1;  // group size 1: no transfer (as k_fused_t)
      const int prevp = j ? (int)(cpos[j - 1] & 0xFFFu) : -1;  // previous comm position of this tile
      // one member: instance record (group leader), wait staged for the flush, sums, edge, stage 2
      auto apply = [&](auto KC, uint32_t mn, uint32_t mx, uint32_t lastrow, uint32_t nat, uint32_t slot, bool lead) {
        constexpr int k = decltype(KC)::value;  // compile-time row block: the register arrays stay registers
        const uint32_t row = lane + 32u * k;
        const uint32_t inst = base[k] + kinst;
        const bool islast = row == lastrow;
        if (lead)
          a.rec[inst] = make_uint4(mn, mx, sbase + lastrow, (SCAN_F_COMPLETE | SCAN_F_KIND_OK | SCAN_F_PAYLOAD_OK | SCAN_F_VALID |
                                                           (nat == 1 ? SCAN_F_UNIQUE_LAST : 0u)) | (clsid << 8));
        const uint32_t wait = d[k] - mn;
        dur_s[wo + 1024u * k] = wait;   // staged for the flush
        comm_s[wo + 1024u * k] = inst;
        acc.wait[k] += wait;
        if (trans) acc.tr[k] += mn;
        if (!islast && (unsigned long long)wait > a.wait_margin) {
          if (win == w_edge) {
            const uint32_t old = atomicAdd(&edge[row * a.ES + slot], wait);
            if (old + wait < old)  // 32-bit wrap: the carry goes straight to the 64-bit global weight
              atomicAdd(&a.ew[(uint64_t)w_edge * a.nnz_tot + a.eidx[(uint64_t)(sbase + row) * E + slot]], 1ull << 32);
          } else {
            atomicAdd(&a.ew[(uint64_t)win * a.nnz_tot + a.eidx[(uint64_t)(sbase + row) * E + slot]], (unsigned long long)wait);
          }
        }
        if (!elig) return;
        bool ps = a.mode != 0;
        if (!ps) ps = seg_any(sbits + row * a.SWD, (uint32_t)(prevp + 1), p) || (prevp < 0 && cflag[row]);
        if (!ps) return;
        if (win != acc.w2) { flush_s2(a, acc, sbase, lane); acc.w2 = win; }
        ++acc.join[k];
        if (islast && nat == 1 && (unsigned long long)(mx - mn) > a.late_margin) ++acc.late[k];
      };
      if (istp) {
        // the NRB TP reductions interleaved (independent shuffle chains), then the members
        uint32_t mnv[NRB], mxv[NRB];
#pragma unroll
        for (int k = 0; k < NRB; ++k) {
          const bool valid = (vmask >> k) & 1u;
          mnv[k] = valid ? d[k] : 0xFFFFFFFFu; mxv[k] = valid ? d[k] : 0u;
        }
        for (uint32_t m = 1; m < TP; m <<= 1)
#pragma unroll
          for (int k = 0; k < NRB; ++k) {
            mnv[k] = min(mnv[k], __shfl_xor_sync(0xFFFFFFFFu, mnv[k], m));
            mxv[k] = max(mxv[k], __shfl_xor_sync(0xFFFFFFFFu, mxv[k], m));
          }
        unsigned eqv[NRB];
#pragma unroll
        for (int k = 0; k < NRB; ++k) eqv[k] = __ballot_sync(0xFFFFFFFFu, ((vmask >> k) & 1u) && d[k] == mnv[k]) & gmt;
        static_for<NRB>([&](auto KC) {
          constexpr int k = decltype(KC)::value;
          const uint32_t ls = eqv[k] ? (uint32_t)(__ffs(eqv[k]) - 1) : 0u;
          if ((vmask >> k) & 1u) apply(KC, mnv[k], mxv[k], ls + 32u * k, __popc(eqv[k]), ls & (TP - 1u), tp == 0);
        });
      } else {
        uint32_t mn = 0xFFFFFFFFu, mx = 0;
#pragma unroll
        for (int k = 0; k < NRB; ++k)
          if ((vmask >> k) & 1u) { mn = min(mn, d[k]); mx = max(mx, d[k]); }
        for (uint32_t m = TP; m < 32; m <<= 1) {
          mn = min(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, m));
          mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, m));
        }
        uint32_t lsd = 0xFFFFFFFFu, nat = 0;  // lowest DP index with the minimum, tie count
#pragma unroll
        for (int k = 0; k < NRB; ++k)
          if (((vmask >> k) & 1u) && d[k] == mn) { lsd = min(lsd, (lane + 32u * k) >> tpsh); ++nat; }
        for (uint32_t m = TP; m < 32; m <<= 1) {
          lsd = min(lsd, __shfl_xor_sync(0xFFFFFFFFu, lsd, m));
          nat += __shfl_xor_sync(0xFFFFFFFFu, nat, m);
        }
        static_for<NRB>([&](auto KC) {
          constexpr int k = decltype(KC)::value;
          if ((vmask >> k) & 1u) apply(KC, mn, mx, tp + (lsd << tpsh), nat, TP + lsd, lane + 32u * k < TP);
        });
      }
    }
    SG_T(4);
    bar_sync(SG_BAR_B);
    SG_T(5);

    // ------------------------------------------------------------------ carry + flush
    if (wid == 0 && (ctl[0] || (a.mode == 0 && glob[0] && cT))) {
      // slow bits of the tile -> the global per-rank bit words (one atomic per word); pslow carried into
      // the next tile (mode 0): slow bits after the tile's last comm position (or, with no comm position,
      // the incoming flag or any slow bit of the tile); then clear the tile's bits
      const bool tbits = ctl[0] != 0;
      const uint32_t lastp = cT ? (cpos[cT - 1] & 0xFFFu) : 0u;
      bool any = false;
      if (tbits && !(a.exp & 8u)) {
        // slow bits of the tile -> the global per-rank bit words (by compute index): lanes over positions,
        // one OR-reduction and one atomic per touched word, for each row holding a slow bit
#pragma unroll
        for (int k = 0; k < NRB; ++k) {
          bool has = false;
          if ((vmask >> k) & 1u)
            for (uint32_t w = 0; w < a.SWD; ++w) has |= sbits[(lane + 32u * k) * a.SWD + w] != 0;
          for (uint32_t hm = __ballot_sync(0xFFFFFFFFu, has); hm; hm &= hm - 1) {
            const uint32_t row = 32u * k + (uint32_t)(__ffs(hm) - 1);
            uint32_t* gb = a.bits + boff[row];
            for (uint32_t c0 = 0; c0 < np; c0 += 32) {
              const uint32_t pp = c0 + lane;
              const bool bit = pp < np && ((sbits[row * a.SWD + (pp >> 5)] >> (pp & 31u)) & 1u);
              const uint32_t jj = j0 + (pp < np ? (pa[pp] & 1023u) : 0u);
              const uint32_t wlo = __reduce_min_sync(0xFFFFFFFFu, bit ? (jj >> 5) : 0xFFFFFFFFu);
              if (wlo == 0xFFFFFFFFu) continue;
              const uint32_t whi = __reduce_max_sync(0xFFFFFFFFu, bit ? (jj >> 5) : 0u);
              for (uint32_t w = wlo; w <= whi; ++w) {
                const uint32_t v = __reduce_or_sync(0xFFFFFFFFu, (bit && (jj >> 5) == w) ? (1u << (jj & 31u)) : 0u);
                if (v && lane == 0) atomicOr(gb + w, v);
              }
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < NRB; ++k) {
        const uint32_t row = lane + 32u * k;
        if (!((vmask >> k) & 1u)) continue;
        uint32_t* rb = sbits + row * a.SWD;
        if (a.mode == 0 && !(a.exp & 16u)) {
          const bool f = cT ? seg_any(rb, lastp + 1, np) : (cflag[row] != 0 || seg_any(rb, 0, np));
          cflag[row] = f ? 1u : 0u;
          any |= f;
        }
        if (tbits) for (uint32_t w = 0; w < a.SWD; ++w) rb[w] = 0;
      }
      any = __any_sync(0xFFFFFFFFu, any);
      __syncwarp();
      if (lane == 0) { if (a.mode == 0) glob[0] = any ? 1u : 0u; ctl[0] = 0; }
    }
    // coalesced per-rank rows of instance ids (every comm event) and waits (TP / DP members; the
    // cross-stage members' waits stay in their slots, k_cross_reduce): flat (row, comm index) pairs
    // over every lane of the consumer warps, consecutive lanes -> consecutive comm events of a row
    SG_T(6);
    if (cT) {
      const uint32_t n = R * cT;
      const uint32_t rcp = (uint32_t)((0x100000000ull + cT - 1) / cT);  // exact for n < 2^22 (as fdiv)
      for (uint32_t i2 = ctid; i2 < n; i2 += 32 * SG_NCW) {
        const uint32_t row = cT == 1 ? i2 : __umulhi(i2, rcp), jj = i2 - row * cT;
        const uint32_t cv = cpos[jj];
        const uint32_t off = (pw(cv & 0xFFFu) ^ ((row & 7u) << 2)) + row * 32u;
        const uint64_t o = coffr[row] + m0 + jj;
        a.inst_c[o] = comm_s[off];
        a.wait_c[o] = (cv >> 12) < 2 ? dur_s[off] : 0u;  // cross: placeholder until k_xwait_scatter
      }
    }
    fence_proxy_async();  // generic-proxy accesses of the slot before the next TMA overwrites it
    __syncwarp();
    if (lane == 0) mbar_arrive(bar0 + 8 * (SG_NS + s));
  }
  // ---- end of the range
  SG_T(7);
  if (prof && lane == 0)
    for (int q = 0; q < 8; ++q) a.dbg[(uint64_t)blockIdx.x * 8 + q] = ph[q];
#undef SG_T
  if (__any_sync(0xFFFFFFFFu, mis) && lane == 0) atomicOr(&a.cnt->overflow, NOT_SPMD);
  bar_sync(SG_BAR_C);
  flush_edges(a, edge, slowc, sbase, w_edge, ctid);
  flush_sums(a, acc, sbase, lane);
  flush_s1(a, acc, sbase, lane);
  flush_s2(a, acc, sbase, lane);
}

// ----------------------------------------------------------------------------- host side
static size_t stage_layout(uint32_t T, uint32_t R, uint32_t TP, uint32_t DP, uint32_t NCRM, uint32_t PP, StageArgs* a) {
  auto al = [](size_t x, size_t b) { return (x + b - 1) & ~(b - 1); };
  // swizzled TMA regions need 1024-byte alignment (the kernel aligns the dynamic base; +1024 below)
  const uint32_t RGN = (uint32_t)al((size_t)R * 128, 1024), KRGN = RGN;
  const uint32_t H = (T + 31) / 32, HK = (T + 63) / 64;
  const uint32_t RSK = 2 * T + 16, SWD = (T + 31) / 32, E = TP + DP, ES = E | 1u, NRT = NCRM + SG_NPR;
  size_t o = 0;
  const uint32_t o_dur = 0;
  o += (size_t)H * RGN;
  const uint32_t o_comm = (uint32_t)o;
  o += (size_t)H * RGN;
  const uint32_t o_kind = (uint32_t)o;
  o = al(o + std::max((size_t)HK * KRGN, (size_t)R * RSK), 128);
  const uint32_t o_pa = (uint32_t)o; o = al(o + (size_t)T * 4, 16);
  const uint32_t o_pb = (uint32_t)o; o = al(o + (size_t)T * 4, 16);
  const uint32_t o_pk = (uint32_t)o; o = al(o + (size_t)T * 2, 16);
  const uint32_t o_tb = (uint32_t)o; o = al(o + SG_TBW * 4, 16);
  const uint32_t o_sb = (uint32_t)o; o = al(o + (size_t)R * SWD * 4, 16);
  const uint32_t o_cpos = (uint32_t)o; o = al(o + (size_t)T * 2, 16);
  const uint32_t o_ctl = (uint32_t)o; o = al(o + 16, 1024);
  const uint32_t stage_bytes = (uint32_t)o;
  o = (size_t)stage_bytes * SG_NS;
  const uint32_t o_bar = (uint32_t)o; o = al(o + 16 * SG_NS, 16);
  const uint32_t o_edge = (uint32_t)o; o = al(o + (size_t)R * ES * 4, 16);
  const uint32_t o_coffr = (uint32_t)o; o = al(o + (size_t)R * 8, 16);
  const uint32_t o_rt = (uint32_t)o; o = al(o + (size_t)R * NRT * 16, 16);
  const uint32_t o_rmap = (uint32_t)o; o = al(o + ROLES, 16);
  const uint32_t o_cflag = (uint32_t)o; o = al(o + (size_t)R * 4, 16);
  const uint32_t o_glob = (uint32_t)o; o = al(o + 16, 16);
  const uint32_t o_st = (uint32_t)o; o = al(o + (size_t)(2 * PP + 1) * 4, 16);
  const uint32_t o_strb = (uint32_t)o; o = al(o + (size_t)PP * 8, 16);
  const uint32_t o_slowc = (uint32_t)o; o = al(o + (size_t)R * 4, 16);
  const uint32_t o_boff = (uint32_t)o; o = al(o + (size_t)R * 8, 16);
  const uint32_t o_rel = (uint32_t)o; o = al(o + 4 * SG_NS, 16);
  if (a) {
    a->RGN = RGN; a->KRGN = KRGN; a->RSK = RSK; a->SWD = SWD; a->ES = ES; a->NRT = NRT;
    a->stage_bytes = stage_bytes; a->o_dur = o_dur; a->o_comm = o_comm; a->o_kind = o_kind; a->o_pa = o_pa; a->o_pb = o_pb;
    a->o_pk = o_pk; a->o_tb = o_tb; a->o_sb = o_sb; a->o_cpos = o_cpos; a->o_ctl = o_ctl;
    a->o_bar = o_bar; a->o_edge = o_edge; a->o_coffr = o_coffr; a->o_rt = o_rt; a->o_rmap = o_rmap; a->o_cflag = o_cflag;
    a->o_glob = o_glob; a->o_st = o_st; a->o_strb = o_strb; a->o_slowc = o_slowc; a->o_boff = o_boff; a->o_rel = o_rel;
  }
  return o + 1024;
}

constexpr size_t SG_SMEM_CAP = 227 * 1024;

// tile size of the persistent kernel for R rows (0 = not applicable): the largest multiple of 64
// positions whose 2-stage ring fits, capped at 1024 (10-bit template fields)
uint32_t stage_tile(uint32_t R, uint32_t TP, uint32_t DP, uint32_t NCRM, uint32_t PP) {
  if (R > 128 || TP > 32 || (32 % TP) != 0) return 0;
  uint32_t best = 0;
  for (uint32_t T = 64; T <= 1024; T += 64)
    if (stage_layout(T, R, TP, DP, NCRM, PP, nullptr) <= SG_SMEM_CAP) best = T;
  return best;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda at link time)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                  const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn f = nullptr;
  if (!f) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
      f = reinterpret_cast<EncodeTiledFn>(p);
  }
  return f;
}

// the per-stage 2-D views {npos, R} of dur / comm / kind, 128-byte swizzle, boxes {128 B, R}; false on failure
static bool build_tmaps(Ctx& c) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return false;
  const uint32_t R = c.FR;
  c.kind2d = true;
  for (int st = 0; st < c.PP; ++st) {
    const uint64_t rb = c.h_rank_off[(size_t)st * R];
    const uint32_t np = c.h_st_npos[st];
    if (np && ((rb % 8) || (np % 8))) c.kind2d = false;
  }
  std::vector<CUtensorMap> maps((size_t)c.PP * 3);
  std::memset(maps.data(), 0, maps.size() * sizeof(CUtensorMap));
  for (int st = 0; st < c.PP; ++st) {
    const uint64_t rb = c.h_rank_off[(size_t)st * R];
    const uint32_t np = c.h_st_npos[st];
    if (!np) continue;
    for (int col = 0; col < 3; ++col) {
      if (col == 2 && !c.kind2d) continue;
      const uint32_t es = col == 2 ? 2 : 4;
      void* base = col == 0 ? (void*)(c.d_dur + rb) : (col == 1 ? (void*)(c.d_comm + rb) : (void*)(c.d_kind + rb));
      const cuuint64_t dims[2] = {np, R};
      const cuuint64_t strides[1] = {(cuuint64_t)np * es};
      const cuuint32_t box[2] = {128u / es, R};
      const cuuint32_t estr[2] = {1, 1};
      const CUresult r = enc(&maps[(size_t)st * 3 + col], col == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 2,
                             base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return false;
    }
  }
  if (c.tmaps.ensure(maps.size() * sizeof(CUtensorMap)) != cudaSuccess) return false;
  if (cudaMemcpyAsync(c.tmaps.p, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice, c.stream) != cudaSuccess)
    return false;
  if (cudaStreamSynchronize(c.stream) != cudaSuccess) return false;  // once per load: the host vector dies here
  c.tmap_load = c.load_id;
  return true;
}

int launch_stage(Ctx& c) {
  if (c.tmap_load != c.load_id && !build_tmaps(c)) return -1;  // caller falls back to the transposed kernel
  StageArgs a{};
  a.tmaps = c.tmaps.as<uint8_t>(); a.kind2d = c.kind2d ? 1 : 0;
  { const char* e = std::getenv("MS_STAGE_EXP"); a.exp = e ? (uint32_t)std::atoi(e) : 0u; }
  static DevBuf dbg;
  a.dbg = nullptr;
  if (a.exp & 64u) { dbg.ensure(148 * 8 * 8 * 4); cudaMemsetAsync(dbg.p, 0, 148 * 8 * 8 * 4, c.stream); a.dbg = dbg.as<unsigned long long>(); }
  a.dur = c.d_dur; a.kind = c.d_kind; a.comm = c.d_comm; a.n_events = c.N;
  a.rank_off = c.rank_off.as<uint64_t>(); a.TP = c.TP; a.DP = c.DP; a.PP = c.PP; a.W = c.W; a.n_comms = c.n_comms;
  a.T = c.FT; a.R = c.FR; a.n_ftiles = c.n_ftiles;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  a.n_cta = std::min<uint32_t>(c.n_ftiles, (uint32_t)sms);
  a.st_tile0 = c.st_tile0.as<uint32_t>(); a.st_npos = c.st_npos.as<uint32_t>(); a.st_tot = c.st_tot.as<uint32_t>();
  a.posA = c.ft_posA.as<uint32_t>(); a.posB = c.ft_posB.as<uint32_t>(); a.posK = c.ft_posK.as<uint16_t>();
  a.tbase = c.ft_tbase.as<uint32_t>();
  a.role_comm = c.role_comm.as<uint32_t>(); a.role_slot = c.role_slot.as<uint32_t>(); a.ncroles = c.ncroles.as<uint32_t>();
  a.role_type = c.role_type.as<uint8_t>(); a.NCRM = c.NCRM; a.eidx = c.eidx.as<uint32_t>(); a.coff = c.coff.as<uint64_t>();
  a.ch_base = c.ch_base.as<uint64_t>(); a.ch_slot = c.ch_slot.as<uint64_t>(); a.bitmap = c.bitmap.as<uint32_t>();
  a.bitpre = c.bitpre.as<uint32_t>(); a.comm_off = c.r_comm_off.as<uint64_t>(); a.comp_off = c.r_comp_off.as<uint64_t>();
  a.bits_off = c.r_bits_off.as<uint64_t>(); a.inst_c = c.inst_c.as<uint32_t>(); a.wait_c = c.wait_c.as<uint32_t>();
  a.bits = c.bits.as<uint32_t>(); a.cref = c.cref.as<uint32_t>(); a.rec = c.inst_rec.as<uint4>();
  a.slots = c.slots.as<uint4>();
  a.p2p_slot0 = c.p2p_slot0; a.p2p_inst0 = c.p2p_inst0; a.citer = c.citer.as<uint32_t>(); a.NIT1 = c.NIT + 1;
  a.nnz_tot = c.nnz_c + (uint64_t)c.W * PCAP;
  a.ew = c.ewc.as<unsigned long long>(); a.rk_sum = c.rk_sum.as<unsigned long long>();
  a.wl_joined = c.wl_joined.as<uint32_t>(); a.wl_late = c.wl_late.as<uint32_t>();
  a.wd_total = c.wd_total.as<uint32_t>(); a.wd_slow = c.wd_slow.as<uint32_t>();
  a.slow_num = c.dcfg.slow_num; a.slow_den = c.dcfg.slow_den; a.slow_margin = c.dcfg.slow_margin_ns;
  a.wi = c.dcfg.window_iters; a.classes = c.lcfg.stage2_classes; a.mode = c.lcfg.stage2_mode;
  a.late_margin = c.lcfg.late_margin_ns; a.wait_margin = c.lcfg.wait_margin_ns; a.want_ref = c.dcfg.want_ref ? 1 : 0;
  a.wi_m = c.dcfg.window_iters > 1 ? (~0ull / c.dcfg.window_iters) + 1ull : 0ull;
  a.it_off = c.it_off;
  a.cnt = c.counters.as<Counters>();
  const size_t sm = stage_layout(c.FT, c.FR, c.TP, c.DP, c.NCRM, c.PP, &a);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kern<<<a.n_cta, SG_NT, sm, c.stream>>>(a);
  };
  const uint32_t nrb = (c.FR + 31) / 32;
  auto go_p = [&](auto tagP) {
    constexpr int PP_ = decltype(tagP)::value;
    if (nrb <= 1) go(k_stage<1, PP_>);
    else if (nrb <= 2) go(k_stage<2, PP_>);
    else go(k_stage<4, PP_>);
  };
  if (c.DP < 2) go_p(std::integral_constant<int, 1>{});
  else if (c.DP <= 2) go_p(std::integral_constant<int, 2>{});
  else if (c.DP <= 4) go_p(std::integral_constant<int, 4>{});
  else if (c.DP <= 8) go_p(std::integral_constant<int, 8>{});
  else if (c.DP <= 16) go_p(std::integral_constant<int, 16>{});
  else go_p(std::integral_constant<int, 32>{});
  if (a.exp & 64u) {  // timing experiment: per-CTA phase cycles of warp 0 (stderr)
    std::vector<unsigned long long> h((size_t)a.n_cta * 8);
    cudaMemcpyAsync(h.data(), dbg.p, h.size() * 8, cudaMemcpyDeviceToHost, c.stream);
    cudaStreamSynchronize(c.stream);
    const char* nm[8] = {"setup", "wait_full", "phaseA", "barA", "phaseB", "barB", "carry", "flush"};
    unsigned long long tot[8] = {0}, mx[8] = {0};
    uint32_t worst = 0; unsigned long long wv = 0;
    for (uint32_t b = 0; b < a.n_cta; ++b) {
      unsigned long long sum = 0;
      for (int q = 0; q < 8; ++q) { tot[q] += h[b * 8 + q]; mx[q] = std::max(mx[q], h[b * 8 + q]); sum += h[b * 8 + q]; }
      if (sum > wv) { wv = sum; worst = b; }
    }
    std::fprintf(stderr, "k_stage phases (cycles, warp 0): ");
    for (int q = 0; q < 8; ++q) std::fprintf(stderr, "%s mean %llu max %llu | ", nm[q], tot[q] / a.n_cta, mx[q]);
    std::fprintf(stderr, "\nworst CTA %u (tiles %u..%u): ", worst, (uint32_t)((uint64_t)worst * a.n_ftiles / a.n_cta),
                 (uint32_t)((uint64_t)(worst + 1) * a.n_ftiles / a.n_cta));
    for (int q = 0; q < 8; ++q) std::fprintf(stderr, "%s %llu ", nm[q], h[worst * 8 + q]);
    std::fprintf(stderr, "\n");
  }
  return 1;
}

}  // namespace ms
