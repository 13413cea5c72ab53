// k_align.cu — NEXT-1 timeline alignment (the members of a synchronous call
// "logically finish at the same moment", which "provides anchor points"; a reference rank, the
// others aligned to it "iteratively"; SPEC S:L243-300 ClockMap; readings AL1-AL6).
//
// After an analysis has matched the instances, every rank's local clock is mapped onto the
// reference rank's:
//   AL1 anchors = ends (start + dur) of a rank's collective events whose instance is VALID
//   AL2 ranks are taken in BFS levels from the reference over "shares a valid collective instance";
//       level-k ranks use members of levels < k only
//   AL3 target = max aligned end over those members; anchor = (local end, target - local end) in
//       program order, an end equal to the previous anchor's skipped; decreasing candidate ends on
//       a rank -> SCAN_E_UNSUPPORTED
//   AL4 offset(t): piecewise linear between anchors, floor((o1-o0)(t-t0)/(t1-t0)) in exact 128-bit
//       integers, constant outside, 0 without anchors
//   AL5 aligned start = start + offset(start); unreached ranks keep their clock (level -1)
//   AL6 residual of a rank = max over its candidates of (instance's max aligned end - own)
// Kernels: candidate ends + member-slot index (one warp per 2048-event tile, as the exports),
// communicator reachability, monotonicity (one CTA per rank), per-level anchors (one CTA per rank:
// block scans keep program order and compact), per-level aligned ends, aligned starts, residuals.
#include <algorithm>
#include <climits>
#include <cstdint>
#include <sstream>
#include "internal.cuh"

namespace ms {
namespace {

constexpr long long AL_NONE = (long long)0x8000000000000000ull;  // INT64_MIN: not a candidate

struct AlArgs {
  const uint32_t* tile_rank; const uint64_t* tile_start; const uint64_t* rank_off; const uint16_t* kind;
  const uint32_t* dur; const int64_t* start; uint64_t N, n_tiles;
  const uint32_t* t_commpre; const uint64_t* r_comm_off;
  const uint32_t* inst_c; const uint4* rec;
  const uint64_t* ch_base; const uint64_t* ch_slot; uint64_t NCH;
  const uint64_t* coff; const uint32_t* cmem;
  long long* tend;   // [n_comm] local end of a candidate (AL1), AL_NONE otherwise
  const uint32_t* vbits;  // one bit per instance: VALID (k_al_vbits; L2-resident, unlike the 16-byte records)
  const uint32_t* nmax;   // per channel: this context's occurrences (a shard's range starts at ch_base)
};

// VALID bit of every instance, packed 32 per word (a dense pass over the records)
__global__ void k_al_vbits(uint64_t n_inst, const uint4* rec, uint32_t* vbits) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool v = i < n_inst && (rec[i].w & SCAN_F_VALID);
  const unsigned bm = __ballot_sync(0xFFFFFFFFu, v);
  if (lane_id() == 0 && i < n_inst) vbits[i >> 5] = bm;
}

// candidate ends (AL1)
__global__ void __launch_bounds__(256) k_al_ends(AlArgs a) {
  const uint64_t tile = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (tile >= a.n_tiles) return;
  const uint32_t lane = lane_id();
  const uint32_t r = a.tile_rank[tile];
  const uint64_t s = a.tile_start[tile];
  const uint64_t e = min(s + (uint64_t)TILE_EV, a.rank_off[r + 1]);
  uint32_t comm_carry = a.t_commpre[tile];
  const uint64_t co = a.r_comm_off[r];
  for (uint64_t base = s & ~7ull; base < e; base += 256) {
    const uint64_t g = base + 8ull * lane;
    uint16_t ko[8];
    load8_u16(a.kind, g, a.N, ko);
    uint32_t valid = 0, commm = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint64_t ev = g + q;
      if (ev < s || ev >= e) continue;
      valid |= 1u << q;
      if (ko[q] & 7u) commm |= 1u << q;
    }
    uint32_t ctot;
    const uint32_t cex = warp_excl_scan(__popc(commm), ctot) + comm_carry;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (!((commm >> q) & 1u)) continue;
      const uint64_t ev = g + q;
      const uint64_t ci = co + cex + __popc(commm & ((1u << q) - 1u));
      const uint32_t k = ko[q] & 7u;
      long long t = AL_NONE;
      if (k >= 1 && k <= 4) {
        const uint32_t inst = a.inst_c[ci];
        if ((a.vbits[inst >> 5] >> (inst & 31)) & 1u) t = (long long)a.start[ev] + (long long)a.dur[ev];
      }
      a.tend[ci] = t;
    }
    comm_carry += ctot;
  }
}

// communicators with at least one valid instance connect their members (AL2)
__global__ void k_al_commflag(uint32_t n_comms, const uint64_t* ch_base, const uint32_t* nmax, const uint4* rec, uint8_t* flag) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_comms) return;
  uint8_t f = 0;
  for (uint64_t i = ch_base[c]; i < ch_base[c] + nmax[c] && !f; ++i) f = (rec[i].w & SCAN_F_VALID) ? 1 : 0;
  flag[c] = f;
}

// block-wide exclusive max of i64 (AL_NONE as identity); total = max over the block
__device__ long long block_excl_max_i64(long long v, long long& total, long long* sm /*[33]*/) {
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
  long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= (uint32_t)o) x = max(x, y);
  }
  if (lane == 31) sm[wid] = x;
  __syncthreads();
  if (wid == 0) {
    long long w = lane < (blockDim.x >> 5) ? sm[lane] : AL_NONE;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xFFFFFFFFu, w, o);
      if (lane >= (uint32_t)o) w = max(w, y);
    }
    sm[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  const long long before_warp = wid ? sm[wid - 1] : AL_NONE;
  long long ex = __shfl_up_sync(0xFFFFFFFFu, x, 1);
  if (lane == 0) ex = AL_NONE;
  total = sm[(blockDim.x >> 5) - 1];
  __syncthreads();
  return max(before_warp, ex);
}

constexpr uint32_t AL_SPLIT = 16;  // CTAs per rank in the per-rank passes (blockIdx.y)
// one segment (1/AL_SPLIT of a rank's candidates) of the split per-rank passes: its first and last
// (largest) end -- in the anchor dedupe only ends with a target, AL_NONE if none -- and its anchors
// counted from an empty carry
struct AlSegStat { long long first, last; unsigned long long cnt; };

// AL3 precondition: candidate ends non-decreasing along each rank's program order (AL_SPLIT CTAs per
// rank, each checks its segment; k_al_mono_bnd checks the segment boundaries)
__global__ void __launch_bounds__(256) k_al_mono(const uint64_t* r_comm_off, const long long* tend, uint32_t* bad_rank,
                                                 AlSegStat* seg) {
  __shared__ long long sm[33];
  __shared__ long long carry, first;
  const uint32_t r = blockIdx.x;
  const uint64_t c0 = r_comm_off[r], c1 = r_comm_off[r + 1];
  const uint64_t per = (c1 - c0 + AL_SPLIT - 1) / AL_SPLIT;
  const uint64_t b0 = c0 + per * blockIdx.y, e0 = min(c1, b0 + per);
  if (threadIdx.x == 0) { carry = AL_NONE; first = AL_NONE; }
  __syncthreads();
  for (uint64_t b = b0; b < e0; b += 256) {
    const uint64_t ci = b + threadIdx.x;
    const long long t = ci < e0 ? tend[ci] : AL_NONE;
    long long tot;
    const long long prev = max(block_excl_max_i64(t, tot, sm), carry);
    if (t != AL_NONE && t < prev) atomicMin(bad_rank, r);
    if (t != AL_NONE && prev == AL_NONE) first = t;  // the segment's first candidate end (one thread)
    __syncthreads();
    if (threadIdx.x == 0) carry = max(carry, tot);
    __syncthreads();
  }
  if (threadIdx.x == 0) seg[(uint64_t)r * AL_SPLIT + blockIdx.y] = AlSegStat{first, carry, 0};
}
// the segments of a rank in order: each one's first end must not be below the earlier ones' largest
__global__ void k_al_mono_bnd(uint32_t W, const AlSegStat* seg, uint32_t* bad_rank) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= W) return;
  long long prev = AL_NONE;
  for (uint32_t j = 0; j < AL_SPLIT; ++j) {
    const AlSegStat st = seg[(uint64_t)r * AL_SPLIT + j];
    if (st.last == AL_NONE) continue;
    if (st.first < prev) atomicMin(bad_rank, r);
    prev = max(prev, st.last);
  }
}

// A rank's anchors as one context sees them: its own list (PlainAnc), or (sharded, BndAnc) its own list
// between the rank's last anchor on an earlier shard and its first anchor on a later one (AL_NONE: none)
struct PlainAnc {
  const long long* at; const long long* ao; uint32_t n;
  __device__ __forceinline__ uint32_t size() const { return n; }
  __device__ __forceinline__ long long t(uint32_t i) const { return at[i]; }
  __device__ __forceinline__ long long o(uint32_t i) const { return ao[i]; }
};
struct BndAnc {
  const long long* at; const long long* ao; uint32_t n;
  long long pt, po, nt, no;
  __device__ __forceinline__ uint32_t size() const { return n + (pt != AL_NONE) + (nt != AL_NONE); }
  __device__ __forceinline__ long long t(uint32_t i) const {
    if (pt != AL_NONE) { if (i == 0) return pt; --i; }
    return i < n ? at[i] : nt;
  }
  __device__ __forceinline__ long long o(uint32_t i) const {
    if (pt != AL_NONE) { if (i == 0) return po; --i; }
    return i < n ? ao[i] : no;
  }
};

// index of the last anchor with t(i) <= t (-1 if none): binary search
template <class A>
__device__ __forceinline__ int32_t al_find(const A& v, long long t) {
  uint32_t lo = 0, hi = v.size();
  while (lo < hi) {
    const uint32_t m = (lo + hi) >> 1;
    if (v.t(m) <= t) lo = m + 1; else hi = m;
  }
  return (int32_t)lo - 1;
}
// floor(num / den), den > 0, exact: a double-precision estimate corrected by 128-bit multiplies (a
// 128-bit division is a long software routine on the GPU); exact division for huge quotients
__device__ __forceinline__ __int128 floor_div128(__int128 num, __int128 den) {
  const double qd = floor((double)num / (double)den);
  if (fabs(qd) > 1e15) {
    __int128 q = num / den;
    if ((num % den) != 0 && num < 0) q -= 1;
    return q;
  }
  __int128 q = (__int128)(long long)qd;
  __int128 r = num - q * den;
  while (r < 0) { q -= 1; r += den; }
  while (r >= den) { q += 1; r -= den; }
  return q;
}
// One anchor interval cached in registers: AL4's floor((o1-o0)(t-t0)/(t1-t0)) is recomputed for every
// event, the interval's constants only when the event leaves it. Mode 1 (|o1-o0| < 2^50, t1-t0 < 2^61):
// a double estimate from a per-interval reciprocal, then the exact remainder in wrapping 64-bit
// arithmetic (the true remainder is within a few t1-t0 of 0, so its low 64 bits are it) and +-1
// corrections -- the same floor as floor_div128 without 128-bit products. Mode 2: floor_div128.
struct AlSeg {
  long long o0, o1, t0, tlo, tn, A, D;  // [tlo, tn) = the interval's times (tlo = t(i), or LLONG_MIN before the first anchor)
  double rD;
  int32_t i;      // -3: none yet
  uint32_t mode;  // 0: constant offset o0, 1: 64-bit exact interpolation, 2: 128-bit interpolation
};
// interval i of a rank with n >= 1 anchors, given t(i), t(i+1) (LLONG_MAX past the last), o(i), o(i+1)
__device__ __forceinline__ void al_seg_set(AlSeg& s, int32_t i, uint32_t n, long long t0, long long tn, long long o0, long long o1) {
  s.i = i; s.tlo = t0; s.tn = tn; s.o0 = o0; s.mode = 0;
  if ((uint32_t)i >= n - 1) return;  // constant after the last anchor
  s.o1 = o1; s.t0 = t0;
  const __int128 A = (__int128)o1 - o0, D = (__int128)tn - t0;
  const __int128 lim = (__int128)1 << 50;
  if (A > -lim && A < lim && D < ((__int128)1 << 61)) {
    s.mode = 1; s.A = (long long)A; s.D = (long long)D; s.rD = 1.0 / (double)s.D;
  } else {
    s.mode = 2;
  }
}
template <class V>
__device__ __forceinline__ void al_seg_load(const V& v, int32_t i, AlSeg& s) {
  const uint32_t n = v.size();  // >= 1
  if (i < 0) {  // before the first anchor: o(0)
    s.i = i; s.mode = 0; s.o0 = v.o(0); s.tlo = LLONG_MIN; s.tn = v.t(0);
    return;
  }
  const bool last = (uint32_t)i + 1 >= n;
  al_seg_set(s, i, n, v.t((uint32_t)i), last ? LLONG_MAX : v.t((uint32_t)i + 1), v.o((uint32_t)i), last ? 0 : v.o((uint32_t)i + 1));
}
__device__ __noinline__ long long al_off128(long long o0, long long o1, long long t0, long long t1, long long t) {  // mode 2 (rare): out of line
  return (long long)((__int128)o0 + floor_div128(((__int128)o1 - o0) * ((__int128)t - t0), (__int128)t1 - t0));
}
__device__ __forceinline__ long long al_seg_off(const AlSeg& s, long long t) {
  if (s.mode == 0) return s.o0;
  if (s.mode == 1) {
    const long long dt = t - s.t0;  // 0 <= dt < D: t lies in [t(i), t(i+1))
    long long q = (long long)floor((double)s.A * (double)dt * s.rD);
    long long r = (long long)((unsigned long long)s.A * (unsigned long long)dt - (unsigned long long)q * (unsigned long long)s.D);
    while (r < 0) { --q; r += s.D; }
    while (r >= s.D) { ++q; r -= s.D; }
    return (long long)((unsigned long long)s.o0 + (unsigned long long)q);
  }
  return al_off128(s.o0, s.o1, s.t0, s.tn, t);
}
// A warp's window of AW consecutive anchors of one rank in shared memory, [w0, w0 + AW) (t = LLONG_MAX,
// o = 0 past the last): anchors are dense (one per ~26 events on C3), so a warp's events span a few
// intervals; lanes search the window (6 shared-memory steps) instead of walking global memory.
constexpr int AW = 64;
__device__ __forceinline__ int32_t al_win_find(const long long* wt, long long t) {  // wt[0] <= t < wt[AW-1]
  int32_t j = 0;
#pragma unroll
  for (int st = AW / 2; st >= 1; st >>= 1)
    if (wt[j + st] <= t) j += st;  // j + st <= AW - 1 and wt[AW-1] > t: never past AW - 2
  return j;
}
// (warp-uniform) make the window cover the warp's times [tmin, tmax] from its interval on, if it does not
template <class V>
__device__ __forceinline__ void al_win_place(const V& v, int32_t& w0, long long* wt, long long* wo, long long tmin, long long tmax) {
  if (w0 >= 0 && tmin >= wt[0] && tmax < wt[AW - 1]) return;
  const int32_t i = (w0 >= 0 && tmin >= wt[0] && tmin < wt[AW - 1]) ? w0 + al_win_find(wt, tmin) : al_find(v, tmin);
  w0 = max(i, 0);
  __syncwarp();
  const int32_t n = (int32_t)v.size();
  const uint32_t lane = lane_id();
#pragma unroll
  for (int h = 0; h < AW / 32; ++h) {
    const int32_t j = w0 + (int32_t)lane + 32 * h;
    wt[lane + 32 * h] = j < n ? v.t((uint32_t)j) : LLONG_MAX;
    wo[lane + 32 * h] = j < n ? v.o((uint32_t)j) : 0;
  }
  __syncwarp();
}
template <class V>
__device__ __noinline__ int32_t al_find_ool(const V v, long long t) { return al_find(v, t); }  // t outside the window (rare): out of line
// offset at t (AL4) for a lane: the cached interval, else the window, else a global search
template <class V>
__device__ __forceinline__ long long al_win_off(const V& v, const long long* wt, const long long* wo, int32_t w0, AlSeg& s, long long t) {
  if (s.i != -3 && t >= s.tlo && t < s.tn) return al_seg_off(s, t);
  const uint32_t n = v.size();
  if (t >= wt[0] && t < wt[AW - 1]) {
    const int32_t j = al_win_find(wt, t);
    al_seg_set(s, w0 + j, n, wt[j], wt[j + 1], wo[j], wo[j + 1]);
  } else {
    al_seg_load(v, al_find_ool(v, t), s);
  }
  return al_seg_off(s, t);
}
// interval of t for a cursor that left interval i: a galloping search forward from i+1 when t moved
// forward, a full search when t decreased (or no interval yet)
template <class V>
__device__ __forceinline__ int32_t al_locate(const V& v, int32_t i, long long tlo, long long t) {
  if (i == -3 || t < tlo) return al_find(v, t);
  const int32_t n = (int32_t)v.size();
  if (i + 1 >= n) return i;
  int32_t lo = i + 1, st = 1, hi = lo + 1;  // t(lo) <= t
  while (hi < n && v.t((uint32_t)hi) <= t) { lo = hi; st <<= 1; hi = lo + st; }
  hi = min(hi, n);
  while (hi - lo > 1) {
    const int32_t m = (lo + hi) >> 1;
    if (v.t((uint32_t)m) <= t) lo = m; else hi = m;
  }
  return lo;
}
// offset at t (AL4) for a lane walking program order: the cached interval, else al_locate
template <class V>
__device__ __forceinline__ long long al_cursor_off(const V& v, AlSeg& s, long long t) {
  if (!(s.i != -3 && t >= s.tlo && t < s.tn)) al_seg_load(v, al_locate(v, s.i, s.tlo, t), s);
  return al_seg_off(s, t);
}
__device__ __forceinline__ long long warp_min_i64(long long x) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) x = min(x, __shfl_xor_sync(0xFFFFFFFFu, x, o));
  return x;
}
__device__ __forceinline__ long long warp_max_i64(long long x) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) x = max(x, __shfl_xor_sync(0xFFFFFFFFu, x, o));
  return x;
}
template <bool SH>
__device__ __forceinline__ auto rank_anchors(const long long* at, const long long* ao, uint32_t n, const long long* bnd, uint32_t r) {
  if constexpr (SH) return BndAnc{at, ao, n, bnd[4 * r], bnd[4 * r + 1], bnd[4 * r + 2], bnd[4 * r + 3]};
  else return PlainAnc{at, ao, n};
}


struct AnchorArgs {
  AlArgs a;
  const uint32_t* ranks;  // ranks of this level
  const int32_t* level; int32_t k;
  const long long* aend;  // aligned ends of earlier levels' candidates
  long long* tgt;         // [n_comm] scratch: target of a candidate, AL_NONE if none
  long long* anc_t; long long* anc_o; uint32_t* nanc;
  const long long* imax;  // per instance: max aligned end over members of levels < k (k_al_imax_add)
  const long long* init;  // sharded: per rank, the largest candidate end with a target on earlier shards (dedupe)
  AlSegStat* seg;         // [ranks of the level][AL_SPLIT] per-segment statistics (k_al_target -> k_al_anchor)
};

// Per valid collective instance: the max aligned end over its members of the levels added so far
// (AL3's target for the members of the next level; every reached member for AL6's residual). The
// levels' ranks scatter their candidates' aligned ends with a 64-bit atomic max (AL_SPLIT CTAs per
// rank), one level at a time as the BFS proceeds; a candidate event then reads its instance's value.
__global__ void k_al_imax_fill(uint64_t n, long long* out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = AL_NONE;
}
__global__ void __launch_bounds__(256) k_al_imax_add(AlArgs a, const uint32_t* ranks, const long long* aend, long long* out) {
  const uint32_t r = ranks[blockIdx.x];
  const uint64_t c0 = a.r_comm_off[r], c1 = a.r_comm_off[r + 1];
  const uint64_t per = (c1 - c0 + AL_SPLIT - 1) / AL_SPLIT;
  const uint64_t b = c0 + per * blockIdx.y, e = min(c1, b + per);
  for (uint64_t ci = b + threadIdx.x; ci < e; ci += blockDim.x)
    if (a.tend[ci] != AL_NONE) atomicMax(&out[a.inst_c[ci]], aend[ci]);
}

// AL3 targets for every candidate of the level-k ranks (AL_SPLIT CTAs per rank, fully parallel): the
// instance's max aligned end over members of lower levels (k_al_imax_add). Each CTA also counts its
// segment's anchors as if no end preceded it, with its first and last end that has a target: the
// candidate ends of a rank are non-decreasing (k_al_mono, job-wide on sharded contexts), so a carry c
// from the earlier segments only removes the segment's first anchor, when its end is <= c.
__global__ void __launch_bounds__(256) k_al_target(AnchorArgs A) {
  const AlArgs& a = A.a;
  __shared__ long long sm[33];
  __shared__ long long run, first;
  __shared__ uint32_t cnt;
  const uint32_t r = A.ranks[blockIdx.x];
  const uint64_t c0 = a.r_comm_off[r], c1 = a.r_comm_off[r + 1];
  const uint64_t per = (c1 - c0 + AL_SPLIT - 1) / AL_SPLIT;
  const uint64_t b = c0 + per * blockIdx.y, e = min(c1, b + per);
  if (threadIdx.x == 0) { run = AL_NONE; first = AL_NONE; cnt = 0; }
  __syncthreads();
  for (uint64_t cb = b; cb < e; cb += blockDim.x) {
    const uint64_t ci = cb + threadIdx.x;
    long long t = AL_NONE;
    if (ci < e) {
      // own rank r is at level k, so the instance value (levels < k) excludes it
      const long long te = a.tend[ci];
      const long long tg = te != AL_NONE ? A.imax[a.inst_c[ci]] : AL_NONE;
      A.tgt[ci] = tg;
      if (tg != AL_NONE) t = te;
    }
    long long tot;
    const long long prev = max(block_excl_max_i64(t, tot, sm), run);
    const bool anc = t != AL_NONE && t > prev;
    const int na = __syncthreads_count(anc);
    if (anc && prev == AL_NONE) first = t;  // the segment's first end with a target (one thread)
    if (threadIdx.x == 0) { run = max(run, tot); cnt += (uint32_t)na; }
    __syncthreads();
  }
  if (threadIdx.x == 0) A.seg[(uint64_t)blockIdx.x * AL_SPLIT + blockIdx.y] = AlSegStat{first, run, cnt};
}

// AL3 anchors of the level-k ranks: AL_SPLIT CTAs per rank, each over its segment; its carry (the
// largest earlier end with a target) and its output offset follow from the earlier segments'
// statistics; program order kept by block scans (dedupe against the previous end, stable compaction)
__global__ void __launch_bounds__(256) k_al_anchor(AnchorArgs A) {
  const AlArgs& a = A.a;
  __shared__ long long sm[33];
  __shared__ uint32_t smu[33];
  __shared__ long long last_t;
  __shared__ uint32_t n_anc;
  const uint32_t r = A.ranks[blockIdx.x];
  const uint64_t c0 = a.r_comm_off[r], c1 = a.r_comm_off[r + 1];
  const uint64_t per = (c1 - c0 + AL_SPLIT - 1) / AL_SPLIT;
  const uint64_t b0 = c0 + per * blockIdx.y, e0 = min(c1, b0 + per);
  if (threadIdx.x == 0) {
    long long carry = A.init ? A.init[r] : AL_NONE;
    uint32_t off = 0;
    for (uint32_t j = 0; j < blockIdx.y; ++j) {
      const AlSegStat st = A.seg[(uint64_t)blockIdx.x * AL_SPLIT + j];
      if (st.last == AL_NONE) continue;
      off += (uint32_t)st.cnt - (st.first <= carry ? 1u : 0u);
      carry = max(carry, st.last);
    }
    last_t = carry; n_anc = off;
  }
  __syncthreads();
  for (uint64_t b = b0; b < e0; b += 256) {
    const uint64_t ci = b + threadIdx.x;
    const long long tg = ci < e0 ? A.tgt[ci] : AL_NONE;
    const bool have = tg != AL_NONE;
    const long long t = have ? a.tend[ci] : AL_NONE;
    long long tot;
    const long long prev = max(block_excl_max_i64(t, tot, sm), last_t);
    const bool anc = have && t > prev;
    uint32_t ntot;
    const uint32_t pos = block_excl_sum<256>(anc ? 1u : 0u, ntot, smu);
    if (anc) {
      A.anc_t[c0 + n_anc + pos] = t;
      A.anc_o[c0 + n_anc + pos] = tg - t;
    }
    __syncthreads();
    if (threadIdx.x == 0) { last_t = max(last_t, tot); n_anc += ntot; }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.y == AL_SPLIT - 1) A.nanc[r] = n_anc;
}

// aligned ends of the candidates of level-k ranks (level 0: the reference, offset 0): one CTA per
// rank; a warp takes 1024-event chunks, lane l the events l, l+32, ... (coalesced), one interval
// search per lane and chunk, then a walk (candidate ends are non-decreasing)
#ifndef MS_EV_MINB
#define MS_EV_MINB 4  // 4 CTAs per SM (64 registers)
#endif
template <bool SH>
__global__ void __launch_bounds__(256, MS_EV_MINB) k_al_eval(const uint32_t* ranks, const uint64_t* r_comm_off, const long long* tend,
                                                 const long long* anc_t, const long long* anc_o, const uint32_t* nanc,
                                                 const long long* bnd, long long* aend) {
  __shared__ long long swt[8][AW], swo[8][AW];
  const uint32_t r = ranks[blockIdx.x];
  const uint64_t c0 = r_comm_off[r], c1 = r_comm_off[r + 1];
  const auto A = rank_anchors<SH>(anc_t + c0, anc_o + c0, nanc[r], bnd, r);
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t part = blockIdx.y, warp_g = part * nw + wid, nwg = nw * gridDim.y;
  long long* wt = swt[wid];
  long long* wo = swo[wid];
  const bool any = A.size() > 0;
  for (uint64_t b = c0 + 1024ull * warp_g; b < c1; b += 1024ull * nwg) {
    AlSeg sg;
    sg.i = -3;
    int32_t w0 = -1;
    for (uint64_t cb = b; cb < min(c1, b + 1024); cb += 32) {  // warp-uniform steps of 32 candidates
      const uint64_t ci = cb + lane;
      const long long t = ci < c1 ? tend[ci] : AL_NONE;
      const bool have = t != AL_NONE;
      if (!any) { if (have) aend[ci] = t; continue; }
      const long long tmin = warp_min_i64(have ? t : LLONG_MAX), tmax = warp_max_i64(have ? t : LLONG_MIN);
      if (tmin == LLONG_MAX) continue;
      al_win_place(A, w0, wt, wo, tmin, tmax);
      if (have) aend[ci] = t + al_win_off(A, wt, wo, w0, sg, t);
    }
  }
}

// AL5: aligned start of every event; one warp per 2048-event tile (rank known), lane l the 8
// consecutive events 8l..8l+7 of every 256; the lane's interval is cached across its events (a
// shared-memory anchor window as in k_al_eval, the 8 loads held in registers, shared-memory staging
// of the loads and stores, a 32-bit interpolation mode: each measured no faster, 7.0-9.0 ms on C3)
#ifndef MS_AP_MINB
#define MS_AP_MINB 4  // 4 CTAs per SM (64 registers): 6.7 -> 6.2 ms on C3
#endif
template <bool SH>
__global__ void __launch_bounds__(256, MS_AP_MINB) k_al_apply(uint64_t n_tiles, const uint32_t* tile_rank, const uint64_t* tile_start,
                                                  const uint64_t* rank_off, const uint64_t* r_comm_off, const int32_t* level,
                                                  const int64_t* start, const long long* anc_t, const long long* anc_o,
                                                  const uint32_t* nanc, const long long* bnd, long long* out) {
  const uint64_t tile = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (tile >= n_tiles) return;
  const uint32_t lane = lane_id();
  const uint32_t r = tile_rank[tile];
  const uint64_t s = tile_start[tile];
  const uint64_t e = min(s + (uint64_t)TILE_EV, rank_off[r + 1]);
  const bool on = level[r] >= 0;
  const uint64_t c0 = r_comm_off[r];
  const auto A = rank_anchors<SH>(anc_t + c0, anc_o + c0, nanc[r], bnd, r);
  const uint32_t n = on ? A.size() : 0u;
  AlSeg sg;
  sg.i = -3;
  for (uint64_t g = s + 8ull * lane; g < e; g += 256) {
    const uint64_t ge = min(g + 8, e);
    for (uint64_t ev = g; ev < ge; ++ev) {
      const long long t = start[ev];
      out[ev] = n ? t + al_cursor_off(A, sg, t) : t;
    }
  }
}

// ---- sharded alignment: per-rank values exchanged between the shards
// first / last candidate end of every rank (non-decreasing along program order, so min / max)
__global__ void __launch_bounds__(256) k_al_firstlast(const uint64_t* r_comm_off, const long long* tend, long long* out) {
  __shared__ long long f, l;
  const uint32_t r = blockIdx.x;
  if (threadIdx.x == 0) { f = LLONG_MAX; l = AL_NONE; }
  __syncthreads();
  long long mn = LLONG_MAX, mx = AL_NONE;
  for (uint64_t ci = r_comm_off[r] + threadIdx.x; ci < r_comm_off[r + 1]; ci += blockDim.x) {
    const long long t = tend[ci];
    if (t != AL_NONE) { mn = min(mn, t); mx = max(mx, t); }
  }
  atomicMin(&f, mn); atomicMax(&l, mx);
  __syncthreads();
  if (threadIdx.x == 0) { out[2 * r] = f == LLONG_MAX ? AL_NONE : f; out[2 * r + 1] = l; }
}

// per level-k rank: the largest end of a candidate that has a target (the anchor dedupe's carry)
__global__ void __launch_bounds__(256) k_al_lastT(const uint32_t* ranks, const uint64_t* r_comm_off, const long long* tend,
                                                  const long long* tgt, long long* out) {
  __shared__ long long l;
  const uint32_t r = ranks[blockIdx.x];
  if (threadIdx.x == 0) l = AL_NONE;
  __syncthreads();
  long long mx = AL_NONE;
  for (uint64_t ci = r_comm_off[r] + threadIdx.x; ci < r_comm_off[r + 1]; ci += blockDim.x)
    if (tgt[ci] != AL_NONE) mx = max(mx, tend[ci]);
  atomicMax(&l, mx);
  __syncthreads();
  if (threadIdx.x == 0) out[r] = l;
}

// per level-k rank: its first and last anchor (t, o), AL_NONE if it has none
__global__ void k_al_bounds(uint32_t n, const uint32_t* ranks, const uint64_t* r_comm_off, const long long* anc_t,
                            const long long* anc_o, const uint32_t* nanc, long long* out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t r = ranks[i];
  const uint64_t c0 = r_comm_off[r];
  const uint32_t m = nanc[r];
  out[4 * r] = m ? anc_t[c0] : AL_NONE; out[4 * r + 1] = m ? anc_o[c0] : 0;
  out[4 * r + 2] = m ? anc_t[c0 + m - 1] : AL_NONE; out[4 * r + 3] = m ? anc_o[c0 + m - 1] : 0;
}

// AL6 residuals: one CTA per reached rank, threads over its comm events
__global__ void __launch_bounds__(256) k_al_residual(AlArgs a, const uint32_t* ranks, const long long* imax,
                                                     const long long* aend, unsigned long long* resid) {
  __shared__ unsigned long long best;
  const uint32_t r = ranks[blockIdx.x];
  if (threadIdx.x == 0) best = 0;
  __syncthreads();
  unsigned long long mine = 0;
  const uint64_t c0 = a.r_comm_off[r], c1 = a.r_comm_off[r + 1], per = (c1 - c0 + AL_SPLIT - 1) / AL_SPLIT;
  const uint64_t b0 = c0 + per * blockIdx.y, e0 = min(c1, b0 + per);
  for (uint64_t ci = b0 + threadIdx.x; ci < e0; ci += blockDim.x) {
    if (a.tend[ci] == AL_NONE) continue;
    const long long fin = imax[a.inst_c[ci]];  // the instance's max aligned end over reached members
    mine = max(mine, (unsigned long long)(fin - aend[ci]));
  }
  if (mine) atomicMax(&best, mine);
  __syncthreads();
  if (threadIdx.x == 0 && best) atomicMax(&resid[r], best);
}

}  // namespace

scan_status align_all(Ctx& c, int32_t ref, scan_align_result* out) {
  const uint64_t W = c.W, nc = c.n_comm;
  CK(c.al_tend.ensure(std::max<uint64_t>(nc, 1) * 8)); CK(c.al_aend.ensure(std::max<uint64_t>(nc, 1) * 8));
  CK(c.al_anct.ensure(std::max<uint64_t>(nc, 1) * 8)); CK(c.al_anco.ensure(std::max<uint64_t>(nc, 1) * 8));
  CK(c.al_level.ensure(W * 4));
  CK(c.al_nanc.ensure(W * 4)); CK(c.al_resid.ensure(W * 8));
  CK(c.al_flag.ensure(((c.n_comms + 3) & ~3u) + 4));  // per-comm flags, then the first bad rank (u32)
  CK(c.al_start.ensure(std::max<uint64_t>(c.N, 1) * 8)); CK(c.al_ranks.ensure(W * 4));
  CK(c.al_tgt.ensure(std::max<uint64_t>(nc, 1) * 8));
  CK(c.al_imax.ensure(std::max<uint64_t>(c.p2p_inst0, 1) * 8));  // collective instances come first
  CK(c.al_vbits.ensure((c.n_inst + 31) / 32 * 4 + 4));
  CK(c.al_seg.ensure(W * AL_SPLIT * sizeof(AlSegStat)));
  if (c.n_shards > 1) {
    CK(c.al_lt.ensure(W * 8)); CK(c.al_init.ensure(W * 8)); CK(c.al_bx.ensure(W * 32)); CK(c.al_bnd.ensure(W * 32));
  }
  AlArgs a{c.tile_rank.as<uint32_t>(), c.tile_start.as<uint64_t>(), c.rank_off.as<uint64_t>(), c.d_kind, c.d_dur, c.d_start,
           c.N, c.n_tiles, c.t_commpre.as<uint32_t>(), c.r_comm_off.as<uint64_t>(), c.inst_c.as<uint32_t>(),
           c.inst_rec.as<uint4>(), c.ch_base.as<uint64_t>(), c.ch_slot.as<uint64_t>(), c.NCH, c.coff.as<uint64_t>(),
           c.cmem.as<uint32_t>(), c.al_tend.as<long long>(), c.al_vbits.as<uint32_t>(), c.ch_nmax.as<uint32_t>()};
  int launches = 0;
  if (c.n_inst)
    launches += timed(c, "k_al_ends", [&] {
      k_al_vbits<<<(unsigned)((c.n_inst + 255) / 256), 256, 0, c.stream>>>(c.n_inst, c.inst_rec.as<uint4>(), c.al_vbits.as<uint32_t>());
      return 1;
    });
  if (c.n_tiles) launches += timed(c, "k_al_ends", [&] { k_al_ends<<<(unsigned)((c.n_tiles + 7) / 8), 256, 0, c.stream>>>(a); return 1; });
  if (c.n_comms)
    launches += timed(c, "k_al_commflag", [&] {
      k_al_commflag<<<(c.n_comms + 255) / 256, 256, 0, c.stream>>>(c.n_comms, c.ch_base.as<uint64_t>(), c.ch_nmax.as<uint32_t>(),
                                                                   c.inst_rec.as<uint4>(), c.al_flag.as<uint8_t>());
      return 1;
    });
  uint32_t* bad = reinterpret_cast<uint32_t*>(c.al_flag.as<uint8_t>() + ((c.n_comms + 3) & ~3u));
  CK(cudaMemsetAsync(bad, 0xFF, 4, c.stream));
  launches += timed(c, "k_al_mono", [&] {
    AlSegStat* seg = reinterpret_cast<AlSegStat*>(c.al_seg.p);
    k_al_mono<<<dim3((unsigned)W, AL_SPLIT), 256, 0, c.stream>>>(c.r_comm_off.as<uint64_t>(), c.al_tend.as<long long>(), bad, seg);
    k_al_mono_bnd<<<(unsigned)((W + 255) / 256), 256, 0, c.stream>>>((uint32_t)W, seg, bad);
    return 2;
  });
  std::vector<uint8_t> flag(c.n_comms + 8);
  uint32_t bad_rank = 0;
  const bool sh = c.n_shards > 1;
  const uint32_t G = (uint32_t)c.n_shards, g = (uint32_t)c.shard;
  // sharded: one all-gather of a per-shard row and the host reductions every shard makes alike
  auto gather = [&](const void* src_dev, size_t n_u32, std::vector<uint32_t>& h) -> scan_status {
    CK(c.al_xs.ensure(n_u32 * 4)); CK(c.al_xr.ensure((size_t)G * n_u32 * 4));
    CK(cudaMemcpyAsync(c.al_xs.p, src_dev, n_u32 * 4, cudaMemcpyDeviceToDevice, c.stream));
    const int xr = xch_allgather(c, c.al_xs.p, c.al_xr.p, n_u32);
    if (xr) { c.err = std::string("alignment exchange: ") + xch_error(xr); return SCAN_E_NCCL; }
    h.resize((size_t)G * n_u32);
    CK(cudaMemcpyAsync(h.data(), c.al_xr.p, h.size() * 4, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    return SCAN_OK;
  };
  auto i64at = [](const std::vector<uint32_t>& h, size_t w) { return (long long)((uint64_t)h[w] | ((uint64_t)h[w + 1] << 32)); };
  scan_status gst;
  if (sh) {
    // flags (padded to words) + first bad rank + per-rank first / last candidate end: communicators
    // with a valid instance on any shard connect their members; ends must not decrease across shards
    const size_t fw = ((size_t)c.n_comms + 3) / 4, fe = (fw + 2) & ~size_t(1);  // i64 part 8-byte aligned
    const size_t rowu = fe + 4 * (size_t)W;
    CK(c.al_row.ensure(rowu * 4));
    CK(cudaMemcpyAsync(c.al_row.p, c.al_flag.p, fw * 4 + 4, cudaMemcpyDeviceToDevice, c.stream));
    k_al_firstlast<<<(unsigned)W, 256, 0, c.stream>>>(c.r_comm_off.as<uint64_t>(), c.al_tend.as<long long>(),
                                                      reinterpret_cast<long long*>(c.al_row.as<uint32_t>() + fe));
    launches += 1;
    std::vector<uint32_t> h;
    if ((gst = gather(c.al_row.p, rowu, h))) return gst;
    bad_rank = NONE32;
    for (uint32_t q = 0; q < G; ++q) {
      const uint8_t* fb = reinterpret_cast<const uint8_t*>(h.data() + (size_t)q * rowu);
      for (uint32_t k = 0; k < c.n_comms; ++k) flag[k] |= fb[k];
      bad_rank = std::min(bad_rank, h[(size_t)q * rowu + fw]);
    }
    for (uint64_t r = 0; r < W; ++r) {
      long long prev = AL_NONE;
      for (uint32_t q = 0; q < G; ++q) {
        const size_t w = (size_t)q * rowu + fe + 4 * r;
        const long long f = i64at(h, w), l = i64at(h, w + 2);
        if (f == AL_NONE) continue;
        if (prev != AL_NONE && f < prev) bad_rank = std::min<uint32_t>(bad_rank, (uint32_t)r);
        prev = l;
      }
    }
  } else {
    if (c.n_comms) CK(cudaMemcpyAsync(flag.data(), c.al_flag.p, c.n_comms, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(&bad_rank, bad, 4, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
  }
  CK(cudaGetLastError());
  if (bad_rank != NONE32) {
    std::ostringstream m;
    m << "timeline alignment: collective end times decrease along the program order of rank " << bad_rank;
    c.err = m.str();
    return SCAN_E_UNSUPPORTED;
  }
  // AL2: BFS levels on the host over the communicators that have a valid instance
  std::vector<int32_t> level(W, -1);
  std::vector<uint32_t> order{(uint32_t)ref};
  level[ref] = 0;
  for (size_t q = 0; q < order.size(); ++q) {
    const uint32_t u = order[q];
    for (uint32_t x = c.h_rcomm_off[u]; x < c.h_rcomm_off[u + 1]; ++x) {
      const uint32_t k = c.h_rcomm[x];
      if (!flag[k]) continue;
      for (uint64_t y = c.h_coff[k]; y < c.h_coff[k + 1]; ++y) {
        const uint32_t v = c.h_cmem[y];
        if (level[v] < 0) { level[v] = level[u] + 1; order.push_back(v); }
      }
    }
  }
  int32_t maxlev = 0;
  for (int32_t l : level) maxlev = std::max(maxlev, l);
  std::vector<uint32_t> by_level;  // ranks grouped by level (ascending)
  std::vector<uint32_t> lvl_off(maxlev + 2, 0);
  for (uint64_t r = 0; r < W; ++r) if (level[r] >= 0) ++lvl_off[level[r] + 1];
  for (int32_t l = 0; l <= maxlev; ++l) lvl_off[l + 1] += lvl_off[l];
  by_level.resize(lvl_off[maxlev + 1]);
  {
    std::vector<uint32_t> fill(lvl_off.begin(), lvl_off.end() - 1);
    for (uint64_t r = 0; r < W; ++r) if (level[r] >= 0) by_level[fill[level[r]]++] = (uint32_t)r;
  }
  scan_status st;
  if ((st = upload(c, c.al_level, level)) || (st = upload(c, c.al_ranks, by_level))) return st;
  CK(cudaMemsetAsync(c.al_nanc.p, 0, W * 4, c.stream));
  CK(cudaMemsetAsync(c.al_resid.p, 0, W * 8, c.stream));
  std::vector<long long> bnd(sh ? 4 * (size_t)W : 0);  // per rank: anchors on the neighbouring shards (sharded)
  for (size_t i = 0; i < bnd.size(); i += 4) { bnd[i] = AL_NONE; bnd[i + 1] = 0; bnd[i + 2] = AL_NONE; bnd[i + 3] = 0; }
  if (sh) CK(cudaMemcpyAsync(c.al_bnd.p, bnd.data(), W * 32, cudaMemcpyHostToDevice, c.stream));
  auto eval = [&](int32_t k) {
    const uint32_t n = lvl_off[k + 1] - lvl_off[k];
    if (nc && n)
      launches += timed(c, "k_al_eval", [&] {
        auto go = [&](auto kern) {
          kern<<<dim3(n, AL_SPLIT), 256, 0, c.stream>>>(c.al_ranks.as<uint32_t>() + lvl_off[k], c.r_comm_off.as<uint64_t>(),
                                                        c.al_tend.as<long long>(), c.al_anct.as<long long>(),
                                                        c.al_anco.as<long long>(), c.al_nanc.as<uint32_t>(),
                                                        c.al_bnd.as<long long>(), c.al_aend.as<long long>());
        };
        if (sh) go(k_al_eval<true>); else go(k_al_eval<false>);
        return 1;
      });
  };
  eval(0);
  // instance maxima over the levels added so far: levels [0, added) scattered into al_imax
  int32_t added = 0;
  auto add_levels = [&](int32_t upto) {
    if (!c.n_comms || !nc) { added = upto; return 0; }
    int l = 0;
    if (added == 0) {
      k_al_imax_fill<<<(unsigned)((c.p2p_inst0 + 255) / 256), 256, 0, c.stream>>>(c.p2p_inst0, c.al_imax.as<long long>());
      ++l;
    }
    const uint32_t n = lvl_off[upto] - lvl_off[added];
    if (n) {
      k_al_imax_add<<<dim3(n, AL_SPLIT), 256, 0, c.stream>>>(a, c.al_ranks.as<uint32_t>() + lvl_off[added], c.al_aend.as<long long>(),
                                                             c.al_imax.as<long long>());
      ++l;
    }
    added = upto;
    return l;
  };
  for (int32_t k = 1; k <= maxlev; ++k) {
    const uint32_t n = lvl_off[k + 1] - lvl_off[k];
    AnchorArgs A{a, c.al_ranks.as<uint32_t>() + lvl_off[k], c.al_level.as<int32_t>(), k, c.al_aend.as<long long>(),
                 c.al_tgt.as<long long>(), c.al_anct.as<long long>(), c.al_anco.as<long long>(), c.al_nanc.as<uint32_t>(),
                 c.al_imax.as<long long>(), nullptr, reinterpret_cast<AlSegStat*>(c.al_seg.p)};
    if (n) {
      launches += timed(c, "k_al_target", [&] {
        const int l = add_levels(k);
        k_al_target<<<dim3(n, AL_SPLIT), 256, 0, c.stream>>>(A);
        return l + 1;
      });
      if (sh) {  // the anchor dedupe carries over from the earlier shards: their largest candidate end
        std::vector<long long> zero(W, AL_NONE);
        CK(cudaMemcpyAsync(c.al_lt.p, zero.data(), W * 8, cudaMemcpyHostToDevice, c.stream));
        k_al_lastT<<<n, 256, 0, c.stream>>>(A.ranks, c.r_comm_off.as<uint64_t>(), c.al_tend.as<long long>(),
                                            c.al_tgt.as<long long>(), c.al_lt.as<long long>());
        std::vector<uint32_t> h;
        if ((gst = gather(c.al_lt.p, 2 * W, h))) return gst;
        std::vector<long long> init(W, AL_NONE);
        for (uint64_t r = 0; r < W; ++r)
          for (uint32_t q = 0; q < g; ++q) init[r] = std::max(init[r], i64at(h, (size_t)q * 2 * W + 2 * r));
        CK(cudaMemcpyAsync(c.al_init.p, init.data(), W * 8, cudaMemcpyHostToDevice, c.stream));
        A.init = c.al_init.as<long long>();
        launches += 1;
      }
      launches += timed(c, "k_al_anchor", [&] { k_al_anchor<<<dim3(n, AL_SPLIT), 256, 0, c.stream>>>(A); return 1; });
    }
    if (sh && n) {  // the level-k ranks' neighbouring anchors on the other shards (interpolation across blocks)
      k_al_bounds<<<(n + 255) / 256, 256, 0, c.stream>>>(n, A.ranks, c.r_comm_off.as<uint64_t>(), c.al_anct.as<long long>(),
                                                         c.al_anco.as<long long>(), c.al_nanc.as<uint32_t>(),
                                                         c.al_bx.as<long long>());
      std::vector<uint32_t> h;
      if ((gst = gather(c.al_bx.p, 8 * W, h))) return gst;
      for (uint32_t i = lvl_off[k]; i < lvl_off[k + 1]; ++i) {
        const uint32_t r = by_level[i];
        long long* b = &bnd[4 * (size_t)r];
        b[0] = AL_NONE; b[1] = 0; b[2] = AL_NONE; b[3] = 0;
        for (int64_t q = (int64_t)g - 1; q >= 0; --q) {  // the last anchor of the nearest earlier shard that has one
          const size_t w = (size_t)q * 8 * W + 8 * (size_t)r;
          if (i64at(h, w + 4) != AL_NONE) { b[0] = i64at(h, w + 4); b[1] = i64at(h, w + 6); break; }
        }
        for (uint32_t q = g + 1; q < G; ++q) {  // the first anchor of the nearest later shard that has one
          const size_t w = (size_t)q * 8 * W + 8 * (size_t)r;
          if (i64at(h, w) != AL_NONE) { b[2] = i64at(h, w); b[3] = i64at(h, w + 2); break; }
        }
      }
      CK(cudaMemcpyAsync(c.al_bnd.p, bnd.data(), W * 32, cudaMemcpyHostToDevice, c.stream));
      CK(cudaStreamSynchronize(c.stream));
      launches += 1;
    }
    eval(k);
  }
  if (c.n_tiles)
    launches += timed(c, "k_al_apply", [&] {
      auto go = [&](auto kern) {
        kern<<<(unsigned)((c.n_tiles + 7) / 8), 256, 0, c.stream>>>(
            c.n_tiles, c.tile_rank.as<uint32_t>(), c.tile_start.as<uint64_t>(), c.rank_off.as<uint64_t>(),
            c.r_comm_off.as<uint64_t>(), c.al_level.as<int32_t>(), c.d_start, c.al_anct.as<long long>(),
            c.al_anco.as<long long>(), c.al_nanc.as<uint32_t>(), c.al_bnd.as<long long>(), c.al_start.as<long long>());
      };
      if (sh) go(k_al_apply<true>); else go(k_al_apply<false>);
      return 1;
    });
  if (nc && !by_level.empty())
    launches += timed(c, "k_al_residual", [&] {
      const int l = add_levels(maxlev + 1);
      k_al_residual<<<dim3((unsigned)by_level.size(), AL_SPLIT), 256, 0, c.stream>>>(a, c.al_ranks.as<uint32_t>(), c.al_imax.as<long long>(),
                                                                     c.al_aend.as<long long>(), c.al_resid.as<unsigned long long>());
      return l + 1;
    });
  std::vector<uint32_t> nanc(W);
  std::vector<uint64_t> resid(W);
  if (sh) {  // job-wide anchor counts (sum) and residuals (max); the exports hold the job's values
    CK(c.al_row.ensure(W * 12));
    CK(cudaMemcpyAsync(c.al_row.p, c.al_nanc.p, W * 4, cudaMemcpyDeviceToDevice, c.stream));
    CK(cudaMemcpyAsync(c.al_row.as<uint32_t>() + W, c.al_resid.p, W * 8, cudaMemcpyDeviceToDevice, c.stream));
    std::vector<uint32_t> h;
    if ((gst = gather(c.al_row.p, 3 * W, h))) return gst;
    for (uint64_t r = 0; r < W; ++r) {
      uint32_t na = 0;
      uint64_t rs = 0;
      for (uint32_t q = 0; q < G; ++q) {
        na += h[(size_t)q * 3 * W + r];
        rs = std::max<uint64_t>(rs, (uint64_t)i64at(h, (size_t)q * 3 * W + W + 2 * r));
      }
      nanc[r] = na; resid[r] = rs;
    }
    CK(cudaMemcpyAsync(c.al_nanc.p, nanc.data(), W * 4, cudaMemcpyHostToDevice, c.stream));
    CK(cudaMemcpyAsync(c.al_resid.p, resid.data(), W * 8, cudaMemcpyHostToDevice, c.stream));
    CK(cudaStreamSynchronize(c.stream));
  } else {
    CK(cudaMemcpyAsync(nanc.data(), c.al_nanc.p, W * 4, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(resid.data(), c.al_resid.p, W * 8, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
  }
  CK(cudaGetLastError());
  resolve_timing(c);
  c.launches += launches;
  if (out) {
    out->n_anchors = 0; out->n_aligned_ranks = 0; out->n_unaligned_ranks = 0; out->max_level = (uint32_t)maxlev;
    out->max_residual_ns = 0;
    for (uint64_t r = 0; r < W; ++r) {
      out->n_anchors += nanc[r];
      if (level[r] >= 0) ++out->n_aligned_ranks; else ++out->n_unaligned_ranks;
      out->max_residual_ns = std::max<uint64_t>(out->max_residual_ns, resid[r]);
    }
  }
  return SCAN_OK;
}

}  // namespace ms
