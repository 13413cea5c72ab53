// k_stats.cu — A4-A8: stage 1 (cross-DP comparison), stage 2 (start lag), stage 3 (P2P
// effective bandwidth), verdicts, wait-for edges and the frontier walk.
//
// PAPER.md P:L139-154; readings R8-R18.
#include <cooperative_groups.h>
#include "internal.cuh"

namespace cg = cooperative_groups;

namespace ms {

// ----------------------------------------------------------------------------- K3 stage 1
// One warp per (peer class, 32 compute positions). Lane = position j. The DP peer durations at j
// are sorted in registers with a bitonic network (padded to P = 2^k with +inf); a = s[q],
// b = s[q+1] with q = floor((dp-2)/2). The leave-one-out lower median of the other dp-1 peers is
// ref_i = (x_i > a) ? a : b  (removing one element below-or-at position q shifts the order
// statistic by one; removing one above it does not; for x_i == a either choice gives b == a or
// the element after the last copy of a — see DESIGN.md §K3).
template <int P>
__device__ __forceinline__ void bitonic_regs(uint32_t (&v)[P]) {
#pragma unroll
  for (int k = 2; k <= P; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const uint32_t x = v[i], y = v[ixj];
          const uint32_t lo = min(x, y), hi = max(x, y);
          v[i] = up ? lo : hi;
          v[ixj] = up ? hi : lo;
        }
      }
}

struct S1Args {
  int TP, PP, DP;
  uint32_t max_chunks;
  const uint64_t* r_comp_off; const uint64_t* r_bits_off;
  const uint32_t* cdur; const uint16_t* cop;
  uint32_t* bits; uint32_t* cref;
  const uint32_t* cl_min; uint32_t* cl_J;
  uint32_t slow_num, slow_den; unsigned long long slow_margin;
};

#ifndef MS_S1_MINB
#define MS_S1_MINB 4  // 4 CTAs per SM (64 registers): 3.9 -> 2.6 ms on C3's general path
#endif
template <int P>
__global__ void __launch_bounds__(256, MS_S1_MINB) k_stage1(S1Args a) {
  const uint64_t wg = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const uint32_t cl = (uint32_t)(wg / a.max_chunks), chunk = (uint32_t)(wg % a.max_chunks);
  if (cl >= (uint32_t)(a.TP * a.PP)) return;
  const uint32_t mincnt = a.cl_min[cl];
  if (chunk * 32u >= mincnt) return;
  const uint32_t lane = lane_id();
  const uint32_t j = chunk * 32u + lane;
  const bool act = j < mincnt;
  const int tp = (int)(cl % (uint32_t)a.TP), pp = (int)(cl / (uint32_t)a.TP);
  uint32_t x[P], s[P];
  uint16_t op0 = 0;
  bool mis = false;
  const int q = (a.DP - 2) / 2;
  const int L = P / 2 - 1 - q;  // low sentinels: s[q], s[q+1] land at fixed indices P/2-1, P/2
#pragma unroll
  for (int d = 0; d < P; ++d) {
    x[d] = 0xFFFFFFFFu;
    if (d < a.DP && act) {
      const uint32_t r = (uint32_t)(tp + a.TP * (d + a.DP * pp));
      const uint64_t off = a.r_comp_off[r] + j;
      x[d] = a.cdur[off];
      const uint16_t op = a.cop[off];
      if (d == 0) op0 = op; else mis |= (op != op0);
    }
    s[d] = d < a.DP ? x[d] : (d < a.DP + L ? 0u : 0xFFFFFFFFu);
  }
  const unsigned mm = __ballot_sync(0xFFFFFFFFu, mis);
  if (mm && lane == 0) atomicMin(&a.cl_J[cl], chunk * 32u + (uint32_t)(__ffs(mm) - 1));
  bitonic_regs<P>(s);
  const uint32_t va = s[P / 2 - 1], vb = s[P / 2];
#pragma unroll
  for (int d = 0; d < P; ++d) {
    if (d >= a.DP) break;
    const uint32_t ref = x[d] > va ? va : vb;
    const unsigned long long du = x[d];
    const bool slow = act && (unsigned long long)a.slow_den * du > (unsigned long long)a.slow_num * ref &&
                      du > (unsigned long long)ref + a.slow_margin;
    const unsigned w = __ballot_sync(0xFFFFFFFFu, slow);
    const uint32_t r = (uint32_t)(tp + a.TP * (d + a.DP * pp));
    if (lane == 0) a.bits[a.r_bits_off[r] + chunk] = w;
    if (a.cref && act) a.cref[a.r_comp_off[r] + j] = ref;
  }
}

__global__ void k_class_counts(int TP, int PP, int DP, const uint32_t* r_ncomp, uint32_t* cl_min, uint32_t* cl_max,
                               uint32_t* cl_J) {
  const int cl = blockIdx.x * blockDim.x + threadIdx.x;
  if (cl >= TP * PP) return;
  const int tp = cl % TP, pp = cl / TP;
  uint32_t mn = 0xFFFFFFFFu, mx = 0;
  for (int d = 0; d < DP; ++d) {
    const uint32_t v = r_ncomp[tp + TP * (d + DP * pp)];
    mn = min(mn, v); mx = max(mx, v);
  }
  if (DP < 2) mn = 0;
  cl_min[cl] = mn; cl_max[cl] = mx; cl_J[cl] = mn;
}

int launch_class_counts(Ctx& c) {
  const int ncl = c.TP * c.PP;
  k_class_counts<<<(ncl + 255) / 256, 256, 0, c.stream>>>(c.TP, c.PP, c.DP, c.r_ncomp.as<uint32_t>(), c.cl_min.as<uint32_t>(),
                                                          c.cl_max.as<uint32_t>(), c.cl_J.as<uint32_t>());
  return 1;
}

int launch_stage1(Ctx& c) {
  const int ncl = c.TP * c.PP;
  launch_class_counts(c);
  if (c.DP < 2 || c.max_ncomp == 0) return 1;
  S1Args a{c.TP, c.PP, c.DP, (c.max_ncomp + 31) / 32, c.r_comp_off.as<uint64_t>(), c.r_bits_off.as<uint64_t>(),
           c.cdur.as<uint32_t>(), c.cop.as<uint16_t>(), c.bits.as<uint32_t>(),
           c.dcfg.want_ref ? c.cref.as<uint32_t>() : nullptr, c.cl_min.as<uint32_t>(), c.cl_J.as<uint32_t>(),
           c.dcfg.slow_num, c.dcfg.slow_den, (unsigned long long)c.dcfg.slow_margin_ns};
  const uint64_t warps = (uint64_t)ncl * a.max_chunks;
  const unsigned blocks = (unsigned)((warps + 7) / 8);
  if (c.DP <= 2) k_stage1<2><<<blocks, 256, 0, c.stream>>>(a);
  else if (c.DP <= 4) k_stage1<4><<<blocks, 256, 0, c.stream>>>(a);
  else if (c.DP <= 8) k_stage1<8><<<blocks, 256, 0, c.stream>>>(a);
  else if (c.DP <= 16) k_stage1<16><<<blocks, 256, 0, c.stream>>>(a);
  else if (c.DP <= 32) k_stage1<32><<<blocks, 256, 0, c.stream>>>(a);
  else return -1;  // dp > 32 unsupported in this build (checked at load)
  return 2;
}

// ----------------------------------------------------------------------------- K4 stage-1 counters
__device__ __forceinline__ uint32_t bits_count(const uint32_t* b, uint32_t lo, uint32_t hi) {
  if (lo >= hi) return 0;
  uint32_t n = 0;
  const uint32_t w0 = lo >> 5, w1 = (hi - 1) >> 5;
  for (uint32_t w = w0; w <= w1; ++w) {
    uint32_t m = b[w];
    if (w == w0) m &= 0xFFFFFFFFu << (lo & 31);
    if (w == w1) m &= 0xFFFFFFFFu >> (31 - ((hi - 1) & 31));
    n += __popc(m);
  }
  return n;
}
__device__ __forceinline__ bool bits_any(const uint32_t* b, uint32_t lo, uint32_t hi) {
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

__device__ __forceinline__ uint32_t iter_start(const uint32_t* citer_r, uint32_t NIT, uint32_t ncomp, uint64_t i) {
  return i > NIT ? ncomp : citer_r[i];
}

// One warp per (window, rank): popcount of the slow bits in the window's compute range, lanes
// striding over the bit words.
__global__ void __launch_bounds__(256) k_stage1_counts(int W, int TP, int DP, uint32_t NW, uint32_t wi, uint32_t NIT,
                                                       const uint32_t* r_ncomp, const uint64_t* r_bits_off,
                                                       const uint32_t* bits, const uint32_t* citer, const uint32_t* cl_J,
                                                       uint32_t* wd_total, uint32_t* wd_slow, uint8_t* wd_cand,
                                                       double* wd_frac, uint32_t cand_num, uint32_t cand_den,
                                                       uint32_t min_samples, Counters* cnt) {
  const uint64_t item = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (item >= (uint64_t)NW * W) return;
  const uint32_t lane = lane_id();
  const uint32_t w = (uint32_t)(item / W), r = (uint32_t)(item % W);
  const uint32_t ncomp = r_ncomp[r];
  uint32_t J = 0;
  if (DP >= 2) {
    const uint32_t cl = (r / (uint32_t)(TP * DP)) * TP + r % TP;
    J = cl_J[cl];
  }
  const uint32_t* citer_r = citer + (uint64_t)r * (NIT + 1);
  uint32_t lo = 0, hi = ncomp;
  if (wi) { lo = iter_start(citer_r, NIT, ncomp, (uint64_t)w * wi); hi = iter_start(citer_r, NIT, ncomp, (uint64_t)(w + 1) * wi); }
  hi = min(hi, J);
  const uint32_t total = hi > lo ? hi - lo : 0;
  uint32_t slow = 0;
  if (total) {
    const uint32_t* b = bits + r_bits_off[r];
    const uint32_t w0 = lo >> 5, w1 = (hi - 1) >> 5;
    for (uint32_t x = w0 + lane; x <= w1; x += 32) {
      uint32_t m = b[x];
      if (x == w0) m &= 0xFFFFFFFFu << (lo & 31);
      if (x == w1) m &= 0xFFFFFFFFu >> (31 - ((hi - 1) & 31));
      slow += __popc(m);
    }
    slow = warp_sum_u32(slow);
  }
  if (lane) return;
  const bool cand = total >= min_samples && (unsigned long long)cand_den * slow > (unsigned long long)cand_num * total;
  wd_total[item] = total; wd_slow[item] = slow; wd_cand[item] = cand ? 1 : 0;
  wd_frac[item] = total ? (double)slow / (double)total : 0.0;
  if (total) atomicAdd(&cnt->n_compared, (unsigned long long)total);
  if (slow) atomicAdd(&cnt->n_slow, (unsigned long long)slow);
  if (cand) atomicAdd(&cnt->n_candidates, 1ull);
}

int launch_stage1_counts(Ctx& c) {
  const uint64_t items = (uint64_t)c.NW * c.W;
  k_stage1_counts<<<(unsigned)((items + 7) / 8), 256, 0, c.stream>>>(
      c.W, c.TP, c.DP, c.NW, c.dcfg.window_iters, c.NIT, c.r_ncomp.as<uint32_t>(), c.r_bits_off.as<uint64_t>(),
      c.bits.as<uint32_t>(), c.citer.as<uint32_t>(), c.cl_J.as<uint32_t>(), c.wd_total.as<uint32_t>(),
      c.wd_slow.as<uint32_t>(), c.wd_cand.as<uint8_t>(), c.wd_frac.as<double>(), c.dcfg.cand_num, c.dcfg.cand_den,
      c.dcfg.min_samples, c.counters.as<Counters>());
  return 1;
}

// ----------------------------------------------------------------------------- K5 event pass
// Third walk of the warp tiles: per comm event wait = dur - dmin (written in comm order),
// per-rank sums, stage-2 joined / late counters (instances whose preceding compute segment holds
// a stage-1 slow op, reading R11), wait-for edge weights (reading R17). Edge weights are combined
// in a per-warp shared-memory hash table and flushed once per tile.
struct EPArgs {
  const uint32_t* tile_rank; const uint64_t* tile_start; const uint64_t* rank_off;
  const uint16_t* kind; const uint32_t* dur; uint64_t N; uint64_t n_tiles; int W, TP, DP;
  const uint32_t* t_commpre; const uint32_t* t_iterpre; const uint32_t* t_prevj;
  const uint64_t* r_comm_off; const uint64_t* r_bits_off;
  const uint32_t* inst_c; const uint4* rec; uint32_t* wait_c;
  const uint32_t* bits; const uint32_t* cl_J;
  const uint64_t* nbc_off; const uint32_t* nbc; const uint32_t* nbp; const uint32_t* nbp_n;
  uint64_t nnz_tot, nnz_c;
  unsigned long long* ew;
  unsigned long long* rk_sum;  // [3][W]
  uint32_t* wl_joined; uint32_t* wl_late;
  uint32_t wi, classes, mode;
  unsigned long long late_margin, wait_margin;
  const uint32_t* order;  // processing order of the tiles (tile_order_ptr), null = index order
};

constexpr int EHT = 32;   // edge hash entries per warp
constexpr int ENB = 128;  // collective neighbours of a rank cached per warp (longer lists: global search)

#ifndef MS_EP_MINB
#define MS_EP_MINB 4  // 4 CTAs per SM (64 registers): 15.5 -> 14.1 ms on C3's general path
#endif
__global__ void __launch_bounds__(256, MS_EP_MINB) k_event_pass(EPArgs a) {
  __shared__ unsigned long long hkey[8][EHT];
  __shared__ unsigned long long hval[8][EHT];
  __shared__ uint32_t snb[8][ENB + PCAP];  // the rank's sorted collective / P2P neighbour lists
  const uint32_t wid = threadIdx.x >> 5;
  uint64_t tile = (uint64_t)blockIdx.x * 8 + wid;
  const uint32_t lane = lane_id();
  hkey[wid][lane] = ~0ull; hval[wid][lane] = 0;
  __syncwarp();
  if (tile >= a.n_tiles) return;
  if (a.order) tile = a.order[tile];
  const uint32_t r = a.tile_rank[tile];
  const uint64_t rstart = a.rank_off[r];
  const uint64_t s = a.tile_start[tile];
  const uint64_t e = min(s + (uint64_t)TILE_EV, a.rank_off[r + 1]);
  uint32_t comm_carry = a.t_commpre[tile], iter_carry = a.t_iterpre[tile];
  int32_t prevj = (int32_t)a.t_prevj[tile];
  const uint64_t comm_off = a.r_comm_off[r];
  const uint32_t* bits_r = a.bits + a.r_bits_off[r];
  uint32_t J = 0;
  if (a.DP >= 2) J = a.cl_J[(r / (uint32_t)(a.TP * a.DP)) * a.TP + r % a.TP];
  const uint32_t w_tile = a.wi ? iter_carry / a.wi : 0;
  uint32_t joined = 0, late = 0;
  unsigned long long s_comp = 0, s_wait = 0, s_tr = 0;
  const uint64_t nb0 = a.nbc_off[r], nb1 = a.nbc_off[r + 1];
  const uint32_t np = a.nbp_n[r];
  // the wait-for edge column search (one per waiting event) on the rank's neighbour lists, staged in
  // shared memory: in global memory the dependent binary-search loads were ~40 % of this kernel
  const uint32_t nnc = (uint32_t)(nb1 - nb0);
  const uint32_t* nbl = nnc <= (uint32_t)ENB ? snb[wid] : a.nbc + nb0;
  for (uint32_t i = lane; i < (uint32_t)ENB; i += 32) if (i < nnc) snb[wid][i] = a.nbc[nb0 + i];
  if (lane < np) snb[wid][ENB + lane] = a.nbp[(uint64_t)r * PCAP + lane];
  __syncwarp();
  for (uint64_t base = s & ~7ull; base < e; base += 256) {
    const uint64_t g = base + 8ull * lane;
    uint16_t ko[8]; uint32_t du[8];
    load8_u16(a.kind, g, a.N, ko);
    load8_u32(a.dur, g, a.N, du);
    uint32_t valid = 0, commm = 0, itm = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint64_t ev = g + q;
      if (ev < s || ev >= e) continue;
      valid |= 1u << q;
      if (ko[q] & 7u) commm |= 1u << q;
      if (ko[q] & 8u) itm |= 1u << q;
    }
    uint32_t ctot, itot;
    const uint32_t cex = warp_excl_scan(__popc(commm), ctot) + comm_carry;
    const uint32_t iex = warp_excl_scan(__popc(itm), itot) + iter_carry;
    // j of this lane's last comm event (j is non-decreasing in program order)
    int32_t mylast = -1;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if ((commm >> q) & 1u) mylast = (int32_t)((uint32_t)(g + q - rstart) - (cex + __popc(commm & ((1u << q) - 1u))));
    const int32_t incmax = warp_incl_max(mylast);
    int32_t exmax = __shfl_up_sync(0xFFFFFFFFu, incmax, 1);
    if (lane == 0) exmax = -1;
    int32_t jprev = max(prevj, exmax);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (!((valid >> q) & 1u)) continue;
      const uint64_t ev = g + q;
      const uint32_t cb = cex + __popc(commm & ((1u << q) - 1u));
      const uint32_t j = (uint32_t)(ev - rstart) - cb;
      if (!((commm >> q) & 1u)) { s_comp += du[q]; continue; }
      const uint32_t inst = a.inst_c[comm_off + cb];
      const uint4 rc = a.rec[inst];
      const uint32_t flags = rc.w & 0xFFu, cls = (rc.w >> 8) & 0xFFu;
      const bool ok = flags & SCAN_F_VALID;
      const uint32_t wait = ok ? du[q] - rc.x : 0u;
      a.wait_c[comm_off + cb] = wait;
      const uint32_t win = a.wi ? (iex + __popc(itm & ((1u << q) - 1u))) / a.wi : 0;
      if (ok) {
        s_wait += wait; s_tr += rc.x;
        if (cls && ((a.classes >> (cls - 1)) & 1u)) {
          const bool pslow = a.mode ? true : bits_any(bits_r, (uint32_t)jprev, min(j, J));
          if (pslow) {
            const bool lt = (flags & SCAN_F_UNIQUE_LAST) && rc.z == r && (unsigned long long)(rc.y - rc.x) > a.late_margin;
            if (win == w_tile) { ++joined; late += lt; }
            else { atomicAdd(&a.wl_joined[(uint64_t)win * a.W + r], 1u); if (lt) atomicAdd(&a.wl_late[(uint64_t)win * a.W + r], 1u); }
          }
        }
        if (rc.z != r && (unsigned long long)wait > a.wait_margin) {
          uint64_t idx;
          const uint32_t pc = lower_bound_u32(nbl, nnc, rc.z);
          if (pc < nnc && nbl[pc] == rc.z) idx = nb0 + pc;
          else idx = a.nnz_c + (uint64_t)r * PCAP + lower_bound_u32(snb[wid] + ENB, np, rc.z);
          const unsigned long long key = (unsigned long long)win * a.nnz_tot + idx;
          uint32_t h = (uint32_t)(key * 0x9E3779B1u) & (EHT - 1);
          bool done = false;
          for (int p = 0; p < EHT && !done; ++p) {
            const unsigned long long old = atomicCAS(&hkey[wid][h], ~0ull, key);
            if (old == ~0ull || old == key) { atomicAdd(&hval[wid][h], (unsigned long long)wait); done = true; }
            h = (h + 1) & (EHT - 1);
          }
          if (!done) atomicAdd(&a.ew[key], (unsigned long long)wait);
        }
      }
      jprev = (int32_t)j;
    }
    comm_carry += ctot;
    iter_carry += itot;
    prevj = max(prevj, __shfl_sync(0xFFFFFFFFu, incmax, 31));
  }
  __syncwarp();
  if (hkey[wid][lane] != ~0ull) atomicAdd(&a.ew[hkey[wid][lane]], hval[wid][lane]);
  s_comp = warp_sum_u64(s_comp); s_wait = warp_sum_u64(s_wait); s_tr = warp_sum_u64(s_tr);
  joined = warp_sum_u32(joined); late = warp_sum_u32(late);
  if (lane == 0) {
    if (s_comp) atomicAdd(&a.rk_sum[r], s_comp);
    if (s_wait) atomicAdd(&a.rk_sum[a.W + r], s_wait);
    if (s_tr) atomicAdd(&a.rk_sum[2 * a.W + r], s_tr);
    if (joined) atomicAdd(&a.wl_joined[(uint64_t)w_tile * a.W + r], joined);
    if (late) atomicAdd(&a.wl_late[(uint64_t)w_tile * a.W + r], late);
  }
}

int launch_event_pass(Ctx& c) {
  if (c.n_tiles == 0) return 0;
  EPArgs a{c.tile_rank.as<uint32_t>(), c.tile_start.as<uint64_t>(), c.rank_off.as<uint64_t>(), c.d_kind, c.d_dur, c.N,
           c.n_tiles, c.W, c.TP, c.DP, c.t_commpre.as<uint32_t>(), c.t_iterpre.as<uint32_t>(), c.t_prevj.as<uint32_t>(),
           c.r_comm_off.as<uint64_t>(), c.r_bits_off.as<uint64_t>(), c.inst_c.as<uint32_t>(), c.inst_rec.as<uint4>(),
           c.wait_c.as<uint32_t>(), c.bits.as<uint32_t>(), c.cl_J.as<uint32_t>(), c.nbc_off.as<uint64_t>(),
           c.nbc.as<uint32_t>(), c.nbp.as<uint32_t>(), c.nbp_n.as<uint32_t>(), c.nnz_c + (uint64_t)c.W * PCAP, c.nnz_c,
           c.ewc.as<unsigned long long>(), c.rk_sum.as<unsigned long long>(), c.wl_joined.as<uint32_t>(),
           c.wl_late.as<uint32_t>(), c.dcfg.window_iters, c.lcfg.stage2_classes, c.lcfg.stage2_mode,
           (unsigned long long)c.lcfg.late_margin_ns, (unsigned long long)c.lcfg.wait_margin_ns, tile_order_ptr(c)};
  k_event_pass<<<(unsigned)((c.n_tiles + 7) / 8), 256, 0, c.stream>>>(a);
  return 1;
}

// ----------------------------------------------------------------------------- K6 link medians
// One CTA per (window, P2P channel): samples = valid instances with transfer > 0 whose SEND lies
// in the window; warm-up samples if >= min_samples (reading R13); lower median under the exact
// order (p/t, instance id) by a shared-memory bitonic sort.
constexpr int LK_NT = 1024;

__device__ __forceinline__ bool samp_less(uint32_t pa, uint32_t ta, uint32_t ia, uint32_t pb, uint32_t tb, uint32_t ib) {
  const unsigned long long l = (unsigned long long)pa * tb, rr = (unsigned long long)pb * ta;
  return l < rr || (l == rr && ia < ib);
}

template <int NT>
__device__ void smem_bitonic(uint32_t* sp, uint32_t* st, uint32_t* si, uint32_t n) {
  uint32_t P = 1;
  while (P < n) P <<= 1;
  for (uint32_t i = n + threadIdx.x; i < P; i += NT) { sp[i] = 0xFFFFFFFFu; st[i] = 1; si[i] = 0xFFFFFFFFu; }
  __syncthreads();
  for (uint32_t k = 2; k <= P; k <<= 1)
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < P; i += NT) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          // element ixj before element i; the padding (index NONE32) after every element, whatever
          // its ratio (a transfer of 0 would otherwise order a pad first)
          const bool gt = si[i] == NONE32 ? si[ixj] != NONE32
                                          : (si[ixj] != NONE32 && samp_less(sp[ixj], st[ixj], si[ixj], sp[i], st[i], si[i]));
          if (gt == up) {
            uint32_t t;
            t = sp[i]; sp[i] = sp[ixj]; sp[ixj] = t;
            t = st[i]; st[i] = st[ixj]; st[ixj] = t;
            t = si[i]; si[i] = si[ixj]; si[ixj] = t;
          }
        }
      }
      __syncthreads();
    }
}

struct LKArgs {
  uint32_t n_comms, n_p2p, NW, wi; int W, TP, DP;
  const uint64_t* ch_base; const uint32_t* ch_nmax; const uint32_t* ch_nmin; const uint32_t* psrc; const uint32_t* pdst;
  const uint4* rec;
  const unsigned long long* key;  // per P2P instance (index i - p2p_inst0): lk_sample_key
  // per P2P instance: payload pay[. * pay_stride] (exact tie order), send iteration iter[. * iter_stride] & it_mask
  const uint32_t* pay; const uint32_t* iter; uint32_t pay_stride, iter_stride, it_mask;
  uint64_t p2p_inst0;
  uint32_t min_samples;
  uint32_t* lk_n; uint8_t* lk_used; uint32_t* lk_medp; uint32_t* lk_medt; double* lk_bw; uint8_t* lk_dir; uint8_t* lk_elig;
  Counters* cnt;
  uint32_t n_shards, shard;  // sharded: this shard computes the links with pid % n_shards == shard
};

constexpr int LM_NT = 256;         // 8 warps, up to 8 CTAs per SM
constexpr int LM_U = 8;            // keys in flight per thread
constexpr uint32_t LM_NB = 2048;   // bins of one selection pass over a key range
constexpr uint32_t LM_CC = 512;    // candidates ranked directly

// warp 0 finds the bin holding rank tgt in an LM_NB-bin histogram (64 bins per lane): (bin, count below it)
__device__ __forceinline__ void hist_find_nb(const uint32_t* hist, uint32_t tgt, uint32_t& bin, uint32_t& below) {
  const uint32_t lane = lane_id();
  const uint4* h4 = reinterpret_cast<const uint4*>(hist + lane * 64);
  uint32_t sum = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) { const uint4 v = h4[i]; sum += v.x + v.y + v.z + v.w; }
  const uint32_t inc = warp_incl_scan(sum), ex = inc - sum;
  const unsigned hit = __ballot_sync(0xFFFFFFFFu, ex <= tgt && tgt < inc);
  if (!hit) {  // tgt beyond the histogram's total (inconsistent inputs): no bin
#ifdef MS_DEBUG_CHECKS
    if (lane == 0) printf("k_link_median: rank %u beyond the histogram total %u (block %u)\n", tgt, __shfl_sync(0xFFFFFFFFu, inc, 31), blockIdx.x);
#endif
    bin = LM_NB; below = 0;
    return;
  }
  const uint32_t L = __ffs(hit) - 1;
  uint32_t acc = __shfl_sync(0xFFFFFFFFu, ex, L), b = 0;
  if (lane == L) {
    for (int i = 0; i < 64; ++i) { const uint32_t v = hist[L * 64 + i]; if (acc + v > tgt) { b = i; break; } acc += v; }
  }
  bin = L * 64 + __shfl_sync(0xFFFFFFFFu, b, L);
  below = __shfl_sync(0xFFFFFFFFu, acc, L);
}

// shared histogram add with the lanes of a warp that share a bin combined (bin >= LM_NB = none)
__device__ __forceinline__ void hist_add(uint32_t* hist, uint32_t bin) {
  const unsigned peers = __match_any_sync(0xFFFFFFFFu, bin);
  if (bin < LM_NB && (lane_id() == (uint32_t)(__ffs(peers) - 1))) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
  for (int o = 16; o > 0; o >>= 1) v = min(v, (unsigned long long)__shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
  for (int o = 16; o > 0; o >>= 1) v = max(v, (unsigned long long)__shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}

// One CTA per (window, link), reading the instances' sample keys (lk_sample_key, written by the
// instance reduction). (1) The window's instances are a contiguous occurrence range (the send
// iteration is nondecreasing in the occurrence index): two binary searches. One pass counts the
// samples (warm-up / all) and their key ranges. (2) Lower-median rank (n-1)/2 of the chosen group
// (warm-up if >= min_samples, reading R13): histogram passes of LM_NB bins over the shrinking key
// range until the target bin holds <= LM_CC samples, which are ranked directly. (3) Ties on the f64
// key: the exact order (p/t, instance index) of reading R13.
__global__ void __launch_bounds__(LM_NT, 4) k_link_median(LKArgs a) {
  // a job the fused pass rejected (the general path reruns it): its inputs are not instance records
  if (*((volatile const unsigned*)&a.cnt->overflow) & NOT_SPMD) return;
  __shared__ __align__(16) uint32_t hist[LM_NB];
  __shared__ unsigned long long cand[LM_CC];
  __shared__ unsigned long long s_min[2], s_max[2], s_lo, s_hi, s_K;
  __shared__ uint32_t s_nw, s_na, s_target, s_cnt, s_nc, s_tg, s_tie, s_pick, s_exact_eq, s_ref, s_k0, s_k1;
  __shared__ uint32_t scan_sm[33];
  __shared__ uint32_t s_bad;
  const uint32_t o = blockIdx.x;
  const uint32_t w = o / a.n_p2p, pid = o % a.n_p2p;
  const uint64_t ch = a.n_comms + pid;
  const uint64_t b = a.ch_base[ch];
  const uint32_t n = a.ch_nmax[ch];
  const uint32_t nmin = a.ch_nmin ? a.ch_nmin[ch] : n;  // samples are valid, hence complete: k < nmin
  const uint32_t tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
  const uint32_t src = a.psrc[pid], dst = a.pdst[pid];
  if (tid == 0) {
    const int dpp = (int)(dst / (uint32_t)(a.TP * a.DP)) - (int)(src / (uint32_t)(a.TP * a.DP));
    a.lk_dir[o] = dpp == 1 ? 0 : (dpp == -1 ? 1 : 2);
    a.lk_n[o] = 0; a.lk_used[o] = 0; a.lk_elig[o] = 0; a.lk_medp[o] = 0; a.lk_medt[o] = 0; a.lk_bw[o] = 0.0;
  }
  if (a.n_shards > 1 && pid % a.n_shards != a.shard) return;  // another shard owns this link: zeros for the all-reduce
  const uint64_t rel0 = b - a.p2p_inst0;
  const unsigned long long* key = a.key + rel0;
  if (tid == 0) {
    uint32_t k0 = 0, k1 = nmin;
    if (a.wi) {  // first k with iteration / wi >= w, then >= w + 1
      auto win = [&](uint32_t k) { return (a.iter[(rel0 + k) * a.iter_stride] & a.it_mask) / a.wi; };
      uint32_t lo = 0, hi = nmin;
      while (lo < hi) { const uint32_t m = (lo + hi) >> 1; if (win(m) < w) lo = m + 1; else hi = m; }
      k0 = lo; hi = nmin;
      while (lo < hi) { const uint32_t m = (lo + hi) >> 1; if (win(m) <= w) lo = m + 1; else hi = m; }
      k1 = lo;
    }
    s_k0 = k0; s_k1 = k1; s_bad = 0;
#ifdef MS_DEBUG_CHECKS
    if (k1 > n || k0 > k1) printf("k_link_median[%u]: range [%u, %u) beyond %u instances (nmin %u)\n", o, k0, k1, n, nmin);
#endif
    s_nw = 0; s_na = 0; s_min[0] = s_min[1] = ~0ull; s_max[0] = s_max[1] = 0;
  }
  __syncthreads();
  const uint32_t k0 = s_k0, k1 = s_k1;
  // (1) counts and key ranges, four loads in flight per thread
  {
    unsigned long long mnw = ~0ull, mxw = 0, mna = ~0ull, mxa = 0;
    uint32_t cw = 0, ca = 0;
    for (uint32_t kb = k0 + tid; kb < k1; kb += LM_U * LM_NT) {
      unsigned long long v[LM_U];
#pragma unroll
      for (int u = 0; u < LM_U; ++u) { const uint32_t k = kb + u * LM_NT; v[u] = k < k1 ? key[k] : LK_NONE; }
#pragma unroll
      for (int u = 0; u < LM_U; ++u) {
        if (v[u] == LK_NONE) continue;
        const unsigned long long kk = v[u] & ~LK_WARM;
        ++ca; mna = min(mna, kk); mxa = max(mxa, kk);
        if (v[u] & LK_WARM) { ++cw; mnw = min(mnw, kk); mxw = max(mxw, kk); }
      }
    }
    cw = warp_sum_u32(cw); ca = warp_sum_u32(ca);
    mnw = warp_min_u64(mnw); mxw = warp_max_u64(mxw); mna = warp_min_u64(mna); mxa = warp_max_u64(mxa);
    if (lane == 0) {
      atomicAdd(&s_nw, cw); atomicAdd(&s_na, ca);
      atomicMin(&s_min[0], mnw); atomicMax(&s_max[0], mxw); atomicMin(&s_min[1], mna); atomicMax(&s_max[1], mxa);
    }
  }
  __syncthreads();
  const uint32_t nw = s_nw;
  const bool use_warm = nw >= a.min_samples;
  const uint32_t nu = use_warm ? nw : s_na;
  if (tid == 0) {
    a.lk_n[o] = nu; a.lk_used[o] = use_warm ? 1 : 0;
    a.lk_elig[o] = nu >= a.min_samples ? 1 : 0;
  }
  if (nu == 0) return;
  // the chosen group's key of instance k, or ~0 (above every key) when k is not in it
  auto gkey = [&](unsigned long long v) -> unsigned long long {
    return (v == LK_NONE || (use_warm && !(v & LK_WARM))) ? ~0ull : (v & ~LK_WARM);
  };
  // (2) lower-median rank over the key range [lo, hi]
  if (tid == 0) { s_lo = s_min[use_warm ? 0 : 1]; s_hi = s_max[use_warm ? 0 : 1]; s_target = (nu - 1) / 2; }
  __syncthreads();
  for (;;) {
    const unsigned long long lo = s_lo, hi = s_hi;
    const uint32_t tgt = s_target;
    if (lo == hi) { if (tid == 0) { s_K = lo; s_tg = tgt; } break; }
    const int sh = max(0, 64 - __clzll((long long)(hi - lo)) - 11);  // (hi - lo) >> sh < LM_NB
    for (uint32_t i = tid; i < LM_NB; i += LM_NT) hist[i] = 0;
    __syncthreads();
    for (uint32_t kb = k0; kb < k1; kb += LM_U * LM_NT) {  // whole warps per round: lanes with one bin add once
      unsigned long long v[LM_U];
#pragma unroll
      for (int u = 0; u < LM_U; ++u) { const uint32_t k = kb + u * LM_NT + tid; v[u] = k < k1 ? gkey(key[k]) : ~0ull; }
#pragma unroll
      for (int u = 0; u < LM_U; ++u)
        hist_add(hist, (v[u] >= lo && v[u] <= hi) ? (uint32_t)((v[u] - lo) >> sh) : LM_NB);
    }
    __syncthreads();
    if (wid == 0) {
      uint32_t bin, below;
      hist_find_nb(hist, tgt, bin, below);
      if (lane == 0 && bin == LM_NB) { s_lo = s_hi = lo; s_cnt = 0; s_nc = 0; s_bad = 1; }
      else if (lane == 0) {
        const unsigned long long nlo = lo + ((unsigned long long)bin << sh);
        s_lo = nlo; s_hi = min(hi, nlo + ((1ull << sh) - 1ull)); s_target = tgt - below; s_cnt = hist[bin]; s_nc = 0;
      }
    }
    __syncthreads();
    if (s_bad) break;
    if (s_lo == s_hi || s_cnt > LM_CC) continue;
    // <= LM_CC samples in [lo, hi]: gather their keys and rank them directly
    const unsigned long long l2 = s_lo, h2 = s_hi;
    for (uint32_t kb = k0; kb < k1; kb += LM_U * LM_NT) {
      unsigned long long vv[LM_U];
#pragma unroll
      for (int u = 0; u < LM_U; ++u) { const uint32_t k = kb + u * LM_NT + tid; vv[u] = k < k1 ? gkey(key[k]) : ~0ull; }
#pragma unroll
      for (int u = 0; u < LM_U; ++u) {
        const unsigned long long v = vv[u];
        const bool c = v >= l2 && v <= h2;
        const unsigned bm = __ballot_sync(0xFFFFFFFFu, c);
        if (!bm) continue;
        uint32_t off = 0;
        if (lane == 0) off = atomicAdd(&s_nc, (uint32_t)__popc(bm));
        off = __shfl_sync(0xFFFFFFFFu, off, 0);
        if (c) cand[off + __popc(bm & ((1u << lane) - 1u))] = v;
      }
    }
    __syncthreads();
    const uint32_t nc = s_nc, t2 = s_target;
#ifdef MS_DEBUG_CHECKS
    if (tid == 0 && (nc > LM_CC || nc != s_cnt)) printf("k_link_median[%u]: %u candidates, histogram said %u\n", o, nc, s_cnt);
#endif
    for (uint32_t j = tid; j < nc; j += LM_NT) {
      const unsigned long long kj = cand[j];
      uint32_t less = 0, eq = 0;
      for (uint32_t q = 0; q < nc; ++q) { const unsigned long long kq = cand[q]; less += kq < kj; eq += kq == kj; }
      if (less <= t2 && t2 < less + eq) { s_K = kj; s_tg = t2 - less; }  // equal keys write equal values
    }
    break;
  }
  __syncthreads();
  if (s_bad) return;  // inconsistent inputs (only on a job the fused pass rejects; the call reruns)
  // (3) tie group = the chosen group's instances with the selected key, ordered by (exact p/t, k)
  const unsigned long long K = s_K;
  const uint32_t tg = s_tg;
  if (tid == 0) { s_tie = 0; s_exact_eq = 1; s_ref = NONE32; s_pick = NONE32; }
  __syncthreads();
  {
    uint32_t nt = 0, first = NONE32;
    for (uint32_t kb = k0 + tid; kb < k1; kb += LM_U * LM_NT) {
      unsigned long long vv[LM_U];
#pragma unroll
      for (int u = 0; u < LM_U; ++u) { const uint32_t k = kb + u * LM_NT; vv[u] = k < k1 ? gkey(key[k]) : ~0ull; }
#pragma unroll
      for (int u = 0; u < LM_U; ++u)
        if (vv[u] == K) { ++nt; first = min(first, kb + u * LM_NT); }
    }
    nt = warp_sum_u32(nt);
    first = __reduce_min_sync(0xFFFFFFFFu, first);
    if (lane == 0 && nt) { atomicAdd(&s_tie, nt); atomicMin(&s_ref, first); }
  }
  __syncthreads();
  auto P_ = [&](uint32_t k) { return a.pay[(rel0 + k) * a.pay_stride]; };
  auto T_ = [&](uint32_t k) { return a.rec[b + k].x; };
#ifdef MS_DEBUG_CHECKS
  if (tid == 0 && (s_tie == 0 || s_ref >= k1)) printf("k_link_median[%u]: tie %u ref %u k1 %u\n", o, s_tie, s_ref, k1);
#endif
  if (s_tie == 0) return;
  if (s_tie == 1) {
    if (tid == 0) s_pick = s_ref;
  } else {
    const uint32_t ref = s_ref;
    const uint32_t pr = P_(ref), tr = T_(ref);
    for (uint32_t k = k0 + tid; k < k1; k += LM_NT)
      if (gkey(key[k]) == K && (unsigned long long)P_(k) * tr != (unsigned long long)pr * T_(k)) s_exact_eq = 0;
    __syncthreads();
    if (s_exact_eq) {
      // one exact ratio: the tg-th tie member in occurrence order (each thread a contiguous chunk of k)
      const uint32_t chunk = (k1 - k0 + LM_NT - 1) / LM_NT;
      const uint32_t c0 = k0 + tid * chunk, c1 = min(k1, c0 + chunk);
      uint32_t cnt = 0;
      for (uint32_t k = c0; k < c1; ++k) cnt += gkey(key[k]) == K;
      uint32_t tot;
      const uint32_t ex = block_excl_sum<LM_NT>(cnt, tot, scan_sm);
      if (ex <= tg && tg < ex + cnt) {
        uint32_t r = tg - ex;
        for (uint32_t k = c0; k < c1; ++k)
          if (gkey(key[k]) == K) { if (r == 0) { s_pick = k; break; } --r; }
      }
    } else {
      // distinct exact ratios behind one f64 value (rare): rank the tie group exactly
      for (uint32_t k = k0 + tid; k < k1; k += LM_NT) {
        if (gkey(key[k]) != K) continue;
        const uint32_t pi = P_(k), ti = T_(k);
        uint32_t rk = 0;
        for (uint32_t j2 = k0; j2 < k1; ++j2)
          if (j2 != k && gkey(key[j2]) == K && samp_less(P_(j2), T_(j2), j2, pi, ti, k)) ++rk;
        if (rk == tg) s_pick = k;
      }
    }
  }
  __syncthreads();
  if (tid == 0 && s_pick != NONE32) {
    const uint32_t pm = P_(s_pick), tm = T_(s_pick);
    if (tm != 0) {  // always, unless the keys and records disagree (a job the fused pass rejects)
      a.lk_medp[o] = pm; a.lk_medt[o] = tm;
      a.lk_bw[o] = (double)pm / (double)tm;
    }
  }
}

// g per (window, direction class) and LinkSlow flags; one CTA per (window, direction class).
__global__ void __launch_bounds__(LK_NT) k_link_flags(uint32_t n_p2p, int W, const uint32_t* psrc, const uint32_t* lk_medp,
                                                      const uint32_t* lk_medt, const uint8_t* lk_dir, const uint8_t* lk_elig,
                                                      uint8_t* lk_slow, uint8_t* wl_link_slow, uint32_t bw_num, uint32_t bw_den,
                                                      Counters* cnt) {
  extern __shared__ uint32_t smem[];
  if (*((volatile const unsigned*)&cnt->overflow) & NOT_SPMD) return;  // rejected by the fused pass (rerun follows)
  uint32_t* sp = smem;
  uint32_t* st = smem + LINK_CAP;
  uint32_t* si = smem + 2 * LINK_CAP;
  __shared__ uint32_t scan_sm[33];
  const uint32_t w = blockIdx.x;
  const uint32_t dir = blockIdx.y;  // one CTA per (window, direction class)
  const uint64_t o0 = (uint64_t)w * n_p2p;
  for (uint32_t i = threadIdx.x; i < n_p2p; i += LK_NT)
    if (lk_dir[o0 + i] == dir) lk_slow[o0 + i] = 0;
  {
    uint32_t carry = 0;
    __syncthreads();
    for (uint32_t kb = 0; kb < n_p2p; kb += LK_NT) {
      const uint32_t l = kb + threadIdx.x;
      const bool sel = l < n_p2p && lk_elig[o0 + l] && lk_dir[o0 + l] == dir;
      uint32_t tot;
      const uint32_t ex = block_excl_sum<LK_NT>(sel ? 1u : 0u, tot, scan_sm);
      if (sel && carry + ex < LINK_CAP) { sp[carry + ex] = lk_medp[o0 + l]; st[carry + ex] = lk_medt[o0 + l]; si[carry + ex] = l; }
      carry += tot;
    }
    __syncthreads();
    if (carry == 0) return;
    if (carry > LINK_CAP) { if (threadIdx.x == 0) atomicOr(&cnt->overflow, 16u); return; }
    smem_bitonic<LK_NT>(sp, st, si, carry);
    const uint32_t m = (carry - 1) / 2;
    const unsigned __int128 pg = sp[m], tg = st[m];
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < carry; i += LK_NT) {
      const unsigned __int128 pl = sp[i], tl = st[i];
      if ((unsigned __int128)bw_den * pl * tg < (unsigned __int128)bw_num * pg * tl) {
        lk_slow[o0 + si[i]] = 1;
        wl_link_slow[(uint64_t)w * W + psrc[si[i]]] = 1;
        atomicAdd(&cnt->n_link_slow, 1ull);
      }
    }
  }
}

// Per-(window, link) medians. Sharded contexts read the job-wide channel tables: the instances of
// an owned link are all present after the shard exchange (shard.cu).
static void link_median_go(Ctx& c, LKArgs& a) {
  k_link_median<<<(unsigned)(c.NW * c.n_p2p), LM_NT, 0, c.stream>>>(a);
}

static LKArgs link_args(Ctx& c) {
  LKArgs a{};
  a.n_comms = c.n_comms; a.n_p2p = (uint32_t)c.n_p2p; a.NW = c.NW; a.wi = c.dcfg.window_iters; a.W = c.W; a.TP = c.TP; a.DP = c.DP;
  a.psrc = c.ch_nsend.as<uint32_t>() + c.n_p2p; a.pdst = c.ch_nrecv.as<uint32_t>() + c.n_p2p;
  a.min_samples = c.lcfg.min_samples; a.lk_n = c.lk_n.as<uint32_t>(); a.lk_used = c.lk_used.as<uint8_t>();
  a.lk_medp = c.lk_medp.as<uint32_t>(); a.lk_medt = c.lk_medt.as<uint32_t>(); a.lk_bw = c.lk_bw.as<double>();
  a.lk_dir = c.lk_dir.as<uint8_t>(); a.lk_elig = c.lk_elig.as<uint8_t>(); a.cnt = c.counters.as<Counters>();
  a.n_shards = 1; a.shard = 0;
  return a;
}

int launch_link_median(Ctx& c) {
  if (c.n_p2p == 0) return 0;
  const bool sh = c.n_shards > 1;
  LKArgs a = link_args(c);
  a.ch_base = (sh ? c.g_base : c.ch_base).as<uint64_t>(); a.ch_nmax = (sh ? c.g_nmax : c.ch_nmax).as<uint32_t>();
  a.ch_nmin = (sh ? c.g_nmin : c.ch_nmin).as<uint32_t>();
  a.rec = c.inst_rec.as<uint4>(); a.key = c.lk_key.as<unsigned long long>();
  // the send slot of P2P instance i is slot p2p_slot0 + 2 (i - p2p_inst0): payload in w, iteration in z
  const uint32_t* sw = reinterpret_cast<const uint32_t*>(c.slots.as<uint4>() + c.p2p_slot0);
  a.pay = sw + 3; a.iter = sw + 2; a.pay_stride = 8; a.iter_stride = 8; a.it_mask = SLOT_IT_MASK;
  a.p2p_inst0 = c.p2p_inst0; a.n_shards = (uint32_t)c.n_shards; a.shard = (uint32_t)c.shard;
  link_median_go(c, a);
  return 1;
}

// Per-link medians over a caller-provided instance layout (streaming: the window's samples in
// link-major, age-minor order; base / nmax indexed by channel id n_comms + pid; instance i's payload
// at pay[2 i], its iteration at iter[i], its sample key at key[i])
int launch_link_median_window(Ctx& c, const uint64_t* base, const uint32_t* nmax, const uint64_t* slot, const uint4* rec,
                              const uint32_t* iter, const uint32_t* pay, const unsigned long long* key, uint64_t n_inst) {
  (void)slot; (void)n_inst;
  if (c.n_p2p == 0) return 0;
  LKArgs a = link_args(c);
  a.ch_base = base; a.ch_nmax = nmax; a.ch_nmin = nullptr; a.rec = rec; a.key = key;
  a.pay = pay; a.iter = iter; a.pay_stride = 2; a.iter_stride = 1; a.it_mask = 0xFFFFFFFFu; a.p2p_inst0 = 0;
  link_median_go(c, a);
  return 1;
}

int launch_link_flags(Ctx& c) {
  if (c.n_p2p == 0) return 0;
  const size_t sm = 3 * LINK_CAP * sizeof(uint32_t);
  cudaFuncSetAttribute(k_link_flags, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_link_flags<<<dim3(c.NW, 3), LK_NT, sm, c.stream>>>((uint32_t)c.n_p2p, c.W, c.ch_nsend.as<uint32_t>() + c.n_p2p,
                                               c.lk_medp.as<uint32_t>(), c.lk_medt.as<uint32_t>(), c.lk_dir.as<uint8_t>(),
                                               c.lk_elig.as<uint8_t>(), c.lk_slow.as<uint8_t>(), c.wl_link_slow.as<uint8_t>(),
                                               c.lcfg.bw_num, c.lcfg.bw_den, c.counters.as<Counters>());
  return 1;
}

int launch_links(Ctx& c) { return launch_link_median(c) + launch_link_flags(c); }

// ----------------------------------------------------------------------------- K7+K8 verdicts + walk
// Cooperative grid: verdicts per (window, rank); roots (ComputeSlow/Both ranks, dst of LinkSlow
// links, lowest (src,dst) first); multi-source BFS over the wait-for edges: at level d+1 every
// unlabelled rank with an edge into level d takes the root of its heaviest such neighbour
// (tie -> smallest rank); leftovers with wait edges are UNATTRIBUTED when the window has a root.
struct WKArgs {
  uint32_t NW; int W; uint32_t n_p2p;
  const uint8_t* wd_cand; const uint32_t* wl_joined; const uint32_t* wl_late; const uint8_t* wl_link_slow;
  uint8_t* wl_verdict; double* wl_frac;
  uint32_t late_num, late_den, min_samples;
  const uint8_t* lk_slow; const uint32_t* psrc; const uint32_t* pdst;
  const uint64_t* nbc_off; const uint32_t* nbc; const uint32_t* nbp; const uint32_t* nbp_n;
  uint64_t nnz_tot, nnz_c;
  const unsigned long long* ew;
  uint8_t* lb_label; uint8_t* lb_rkind; uint32_t* lb_rrank; uint32_t* lb_rsrc; uint32_t* lb_depth;
  unsigned long long* lb_twait;
  int32_t* level; uint32_t* linkroot; uint32_t* nroots; unsigned int* changed;
  Counters* cnt;
};

__global__ void k_walk(WKArgs a) {
  cg::grid_group grid = cg::this_grid();
  if (*((volatile const unsigned*)&a.cnt->overflow) & NOT_SPMD) return;  // every block: rejected job, rerun follows
  const uint64_t items = (uint64_t)a.NW * a.W;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // verdicts and rank roots
  for (uint64_t it = t0; it < items; it += stride) {
    const uint32_t joined = a.wl_joined[it], late = a.wl_late[it];
    a.wl_frac[it] = joined ? (double)late / (double)joined : 0.0;
    int v = SCAN_V_NONE;
    if (a.wd_cand[it]) {
      if (joined < a.min_samples) v = SCAN_V_INSUFFICIENT;
      else if ((unsigned long long)a.late_den * late >= (unsigned long long)a.late_num * joined) v = SCAN_V_COMPUTE_SLOW;
      else v = SCAN_V_EXONERATED;
    }
    if (a.wl_link_slow[it]) v = v == SCAN_V_COMPUTE_SLOW ? SCAN_V_BOTH : SCAN_V_LINK_SLOW;
    a.wl_verdict[it] = (uint8_t)v;
    atomicAdd(&a.cnt->v_count[v], 1ull);
    const uint32_t r = (uint32_t)(it % a.W);
    a.linkroot[it] = NONE32;
    a.lb_rrank[it] = NONE32; a.lb_rsrc[it] = NONE32; a.lb_depth[it] = 0; a.lb_rkind[it] = 0;
    if (v == SCAN_V_COMPUTE_SLOW || v == SCAN_V_BOTH) {
      a.level[it] = 0; a.lb_label[it] = SCAN_L_SOURCE_RANK; a.lb_rkind[it] = 1; a.lb_rrank[it] = r; a.lb_rsrc[it] = r;
      atomicAdd(&a.nroots[it / a.W], 1u);
    } else {
      a.level[it] = -1; a.lb_label[it] = SCAN_L_CLEAN;
    }
  }
  // total wait of every item (sum of its out-edge weights): one warp per item, lanes over neighbours
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t wstride = stride >> 5, wg = t0 >> 5;
  for (uint64_t it = wg; it < items; it += wstride) {
    const uint32_t w = (uint32_t)(it / a.W), r = (uint32_t)(it % a.W);
    const unsigned long long* eww = a.ew + (uint64_t)w * a.nnz_tot;
    unsigned long long tw = 0;
    for (uint64_t q = a.nbc_off[r] + lane; q < a.nbc_off[r + 1]; q += 32) tw += eww[q];
    if (lane < a.nbp_n[r]) tw += eww[a.nnz_c + (uint64_t)r * PCAP + lane];
    tw = warp_sum_u64(tw);
    if (lane == 0) a.lb_twait[it] = tw;
  }
  grid.sync();
  for (uint64_t o = t0; o < (uint64_t)a.NW * a.n_p2p; o += stride)
    if (a.lk_slow[o]) {
      const uint32_t w = (uint32_t)(o / a.n_p2p), pid = (uint32_t)(o % a.n_p2p);
      atomicMin(&a.linkroot[(uint64_t)w * a.W + a.pdst[pid]], pid);
    }
  grid.sync();
  for (uint64_t it = t0; it < items; it += stride)
    if (a.level[it] < 0 && a.linkroot[it] != NONE32) {
      const uint32_t pid = a.linkroot[it];
      a.level[it] = 0; a.lb_label[it] = SCAN_L_SOURCE_LINK; a.lb_rkind[it] = 2;
      a.lb_rrank[it] = (uint32_t)(it % a.W); a.lb_rsrc[it] = a.psrc[pid];
      atomicAdd(&a.nroots[it / a.W], 1u);
    }
  grid.sync();
  for (int d = 0;; ++d) {
    // one warp per unlabelled item: lanes over its neighbours, warp argmax (heaviest edge into
    // level d, ties -> smallest rank)
    for (uint64_t it = wg; it < items; it += wstride) {
      if (a.level[it] >= 0) continue;
      const uint32_t w = (uint32_t)(it / a.W), u = (uint32_t)(it % a.W);
      const uint64_t lw = (uint64_t)w * a.W;
      const unsigned long long* eww = a.ew + (uint64_t)w * a.nnz_tot;
      uint32_t best = NONE32; unsigned long long bw = 0;
      auto take = [&](uint32_t v, unsigned long long x) {
        if (v != NONE32 && (best == NONE32 || x > bw || (x == bw && v < best))) { best = v; bw = x; }
      };
      for (uint64_t q = a.nbc_off[u] + lane; q < a.nbc_off[u + 1]; q += 32) {
        const unsigned long long x = eww[q];
        if (x && a.level[lw + a.nbc[q]] == d) take(a.nbc[q], x);
      }
      if (lane < a.nbp_n[u]) {
        const unsigned long long x = eww[a.nnz_c + (uint64_t)u * PCAP + lane];
        const uint32_t v = a.nbp[(uint64_t)u * PCAP + lane];
        if (x && a.level[lw + v] == d) take(v, x);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint32_t ov = __shfl_xor_sync(0xFFFFFFFFu, best, o);
        const unsigned long long ox = __shfl_xor_sync(0xFFFFFFFFu, bw, o);
        take(ov, ox);
      }
      if (lane == 0 && best != NONE32) {
        a.level[it] = d + 1;
        a.lb_label[it] = SCAN_L_VICTIM;
        a.lb_rkind[it] = a.lb_rkind[lw + best];
        a.lb_rrank[it] = a.lb_rrank[lw + best];
        a.lb_rsrc[it] = a.lb_rsrc[lw + best];
        a.lb_depth[it] = (uint32_t)(d + 1);
        atomicAdd(&a.changed[d & 1], 1u);
      }
    }
    grid.sync();
    const unsigned ch = *((volatile unsigned*)&a.changed[d & 1]);
    if (t0 == 0) a.changed[(d + 1) & 1] = 0;
    grid.sync();
    if (ch == 0) break;
  }
  for (uint64_t it = t0; it < items; it += stride) {
    if (a.level[it] < 0 && a.lb_twait[it] > 0 && a.nroots[it / a.W] > 0) a.lb_label[it] = SCAN_L_UNATTRIBUTED;
    const uint8_t lb = a.lb_label[it];
    if (lb == SCAN_L_SOURCE_RANK || lb == SCAN_L_SOURCE_LINK) atomicAdd(&a.cnt->n_roots, 1ull);
    else if (lb == SCAN_L_VICTIM) atomicAdd(&a.cnt->n_victims, 1ull);
    else if (lb == SCAN_L_UNATTRIBUTED) atomicAdd(&a.cnt->n_unattributed, 1ull);
  }
}

int launch_verdict_walk(Ctx& c) {
  WKArgs a{c.NW, c.W, (uint32_t)c.n_p2p, c.wd_cand.as<uint8_t>(), c.wl_joined.as<uint32_t>(), c.wl_late.as<uint32_t>(),
           c.wl_link_slow.as<uint8_t>(), c.wl_verdict.as<uint8_t>(), c.wl_frac.as<double>(), c.lcfg.late_num,
           c.lcfg.late_den, c.lcfg.min_samples, c.lk_slow.as<uint8_t>(), c.ch_nsend.as<uint32_t>() + c.n_p2p,
           c.ch_nrecv.as<uint32_t>() + c.n_p2p, c.nbc_off.as<uint64_t>(), c.nbc.as<uint32_t>(), c.nbp.as<uint32_t>(),
           c.nbp_n.as<uint32_t>(), c.nnz_c + (uint64_t)c.W * PCAP, c.nnz_c, c.ewc.as<unsigned long long>(),
           c.lb_label.as<uint8_t>(), c.lb_rkind.as<uint8_t>(), c.lb_rrank.as<uint32_t>(), c.lb_rsrc.as<uint32_t>(),
           c.lb_depth.as<uint32_t>(), c.lb_twait.as<unsigned long long>(),
           c.scratch.as<int32_t>(), c.scratch.as<uint32_t>() + (uint64_t)c.NW * c.W,
           c.scratch.as<uint32_t>() + 2ull * c.NW * c.W, c.scratch.as<uint32_t>() + 2ull * c.NW * c.W + c.NW,
           c.counters.as<Counters>()};
  const uint64_t items = (uint64_t)c.NW * c.W;
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_walk, 256, 0);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  int blocks = (int)std::min<uint64_t>((items * 32 + 255) / 256, (uint64_t)std::max(1, nb) * sms);  // a warp per item
  blocks = std::max(blocks, 1);
  void* args[] = {&a};
  cudaLaunchCooperativeKernel((void*)k_walk, blocks, 256, args, 0, c.stream);
  return 1;
}

}  // namespace ms
