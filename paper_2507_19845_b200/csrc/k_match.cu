// k_match.cu — A1-A3: per-rank sequence numbers, instance ids, group-by, timing decomposition.
//
// PAPER.md P:L127-131 ("a single pass over the events then matches those that belong to the
// same communication instance") and P:L133 (members "logically finish at the same moment").
// Readings R2-R6 of DESIGN.md: per-communicator occurrence counter, FIFO per directed P2P pair,
// complete iff k < min member count, wait = dur - dmin, transfer = dmin, last arriver = lowest
// member slot with dur = dmin.
//
// Layout (DESIGN.md §HBM layout): events are processed in warp tiles of TILE_EV consecutive
// events of one rank; every lane owns 8 consecutive events of a 256-event round and loads them
// with 16-byte vector loads. The group-by is a direct-addressed scatter to
// slot(channel, k, member) = slot_base(channel) + k*|members| + member (a one-digit counting
// sort: the instance id is known before the scatter), not a general radix sort.
#include "internal.cuh"

namespace ms {

struct TileArgs {
  const uint32_t* tile_rank; const uint64_t* tile_start; const uint64_t* rank_off;
  const uint16_t* kind; const uint32_t* comm; const uint32_t* dur; const uint16_t* meta; const uint32_t* pay;
  uint64_t N; uint64_t n_tiles; int W; uint32_t n_comms;
  const uint64_t* coff; const uint32_t* cmem;
  Counters* cnt;
  const uint32_t* order;  // processing order of the tiles (tile_order_ptr), null = index order
};

__device__ __forceinline__ bool is_member(const uint64_t* coff, const uint32_t* cmem, uint32_t c, uint32_t r) {
  uint64_t b = coff[c], e = coff[c + 1];
  uint32_t n = (uint32_t)(e - b);
  uint32_t p = lower_bound_u32(cmem + b, n, r);
  return p < n && cmem[b + p] == r;
}

// ----------------------------------------------------------------------------- K1a tile scan
// Per warp tile: schema validation, distinct channel keys with their counts, comm / iter_end
// counts and the offset of the last comm event.
__global__ void __launch_bounds__(256) k_tile_scan(TileArgs a, uint32_t* t_nkeys, uint32_t* t_keys, uint32_t* t_cnt,
                                                    uint32_t* t_ncomm, uint32_t* t_niter, int32_t* t_last) {
  const uint64_t tile = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (tile >= a.n_tiles) return;
  const uint32_t lane = lane_id();
  const uint32_t r = a.tile_rank[tile];
  const uint64_t s = a.tile_start[tile];
  const uint64_t e = min(s + (uint64_t)TILE_EV, a.rank_off[r + 1]);
  uint32_t tkey = NONE32, tcnt = 0, nkeys = 0, ncomm = 0, niter = 0;
  int32_t last = -1;
  bool overflow = false;
  unsigned long long bad = ~0ull;
  for (uint64_t base = s & ~7ull; base < e; base += 256) {
    const uint64_t g = base + 8ull * lane;
    uint16_t ko[8]; uint32_t cm[8];
    load8_u16(a.kind, g, a.N, ko);
    load8_u32(a.comm, g, a.N, cm);
    uint32_t keys[8];
    uint32_t pending = 0, itm = 0;
    int32_t mylast = -1;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint64_t ev = g + q;
      keys[q] = 0;
      if (ev < s || ev >= e) continue;
      const uint32_t kind = ko[q] & 7u;
      if (ko[q] & 8u) itm |= 1u << q;
      if (kind == 0) continue;
      bool ok = true;
      uint32_t key = 0;
      if (kind <= 4) {
        ok = cm[q] < a.n_comms && is_member(a.coff, a.cmem, cm[q], r);
        key = cm[q];
      } else if (kind <= 6) {
        ok = cm[q] < (uint32_t)a.W && cm[q] != r;
        key = a.n_comms + (kind == 5 ? r * (uint32_t)a.W + cm[q] : cm[q] * (uint32_t)a.W + r);
      } else {
        ok = false;
      }
      if (!ok) { bad = min(bad, (unsigned long long)ev); continue; }
      keys[q] = key;
      pending |= 1u << q;
      mylast = (int32_t)(ev - s);
    }
    ncomm += warp_sum_u32(__popc(pending));
    niter += warp_sum_u32(__popc(itm));
    const int32_t round_last = (int32_t)__reduce_max_sync(0xFFFFFFFFu, (unsigned)(mylast + 1)) - 1;
    last = max(last, round_last);
    // count per distinct key (one iteration per distinct key in this round)
    while (__any_sync(0xFFFFFFFFu, pending != 0)) {
      const uint32_t leader = __ffs(__ballot_sync(0xFFFFFFFFu, pending != 0)) - 1;
      uint32_t mykey = 0;
      const int first = __ffs(pending) - 1;
#pragma unroll
      for (int q = 0; q < 8; ++q) if (q == first) mykey = keys[q];
      const uint32_t kappa = __shfl_sync(0xFFFFFFFFu, mykey, leader);
      uint32_t m = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) if (((pending >> q) & 1u) && keys[q] == kappa) m |= 1u << q;
      pending &= ~m;
      const uint32_t tot = warp_sum_u32(__popc(m));
      const uint32_t found = __ballot_sync(0xFFFFFFFFu, tkey == kappa);
      if (found) {
        if (lane == (uint32_t)(__ffs(found) - 1)) tcnt += tot;
      } else if (nkeys < KCAP) {
        if (lane == nkeys) { tkey = kappa; tcnt = tot; }
        ++nkeys;
      } else {
        overflow = true;
      }
    }
  }
  if (bad != ~0ull) atomicMin(&a.cnt->bad_event, bad);
  if (overflow && lane == 0) atomicOr(&a.cnt->overflow, 1u);
  if (lane < nkeys) { t_keys[tile * KCAP + lane] = tkey; t_cnt[tile * KCAP + lane] = tcnt; }
  if (lane == 0) { t_nkeys[tile] = nkeys; t_ncomm[tile] = ncomm; t_niter[tile] = niter; t_last[tile] = last; }
}

int launch_tile_scan(Ctx& c) {
  TileArgs a{c.tile_rank.as<uint32_t>(), c.tile_start.as<uint64_t>(), c.rank_off.as<uint64_t>(), c.d_kind, c.d_comm,
             c.d_dur, c.d_meta, c.d_pay, c.N, c.n_tiles, c.W, c.n_comms, c.coff.as<uint64_t>(), c.cmem.as<uint32_t>(),
             c.counters.as<Counters>()};
  if (c.n_tiles == 0) return 0;
  unsigned blocks = (unsigned)((c.n_tiles + 7) / 8);
  k_tile_scan<<<blocks, 256, 0, c.stream>>>(a, c.t_nkeys.as<uint32_t>(), c.t_keys.as<uint32_t>(), c.t_cnt.as<uint32_t>(),
                                             c.t_ncomm.as<uint32_t>(), c.t_niter.as<uint32_t>(), c.t_last.as<int32_t>());
  return 1;
}

// ----------------------------------------------------------------------------- K1b rank scan
// One CTA per rank: union of the rank's channel keys (sorted = channel order), per tile
// exclusive prefix per key, tile prefixes of comm / iter_end counts and of the compute index of
// the previous comm event, per-rank totals, member-count extremes per communicator, P2P bitmap.
struct RankArgs {
  const uint32_t* rank_tile0; const uint64_t* rank_off; const uint64_t* tile_start;
  const uint32_t* t_nkeys; const uint32_t* t_keys; const uint32_t* t_cnt; uint32_t* t_pref;
  const uint32_t* t_ncomm; const uint32_t* t_niter; const int32_t* t_last;
  uint32_t* t_commpre; uint32_t* t_iterpre; uint32_t* t_prevj;
  uint32_t* r_nkeys; uint32_t* r_keys; uint32_t* r_cnt; uint32_t* r_ncomm; uint32_t* r_niter; uint32_t* r_ncomp;
  const uint32_t* rcomm_off; const uint32_t* rcomm;
  uint32_t* ch_nmax; uint32_t* ch_nmin; uint32_t* bitmap;
  uint32_t* nbp; uint32_t* nbp_n;
  const uint16_t* kind;
  int W; uint32_t n_comms;
  Counters* cnt;
};

constexpr int RS_NT = 256;
constexpr int HASH = 2048;

__global__ void __launch_bounds__(RS_NT) k_rank_scan(RankArgs a) {
  __shared__ uint32_t hset[HASH];
  __shared__ uint32_t skeys[RCAP];
  __shared__ uint32_t scarry[RCAP];
  __shared__ uint32_t tl_keys[RS_NT * 8];   // chunk cache of tile key lists (first 8 keys inline)
  __shared__ uint32_t scan_sm[33];
  __shared__ int32_t scan_smi[33];
  __shared__ uint32_t nk;
  __shared__ uint32_t speer[PCAP * 2];
  __shared__ uint32_t npeer;
  const uint32_t r = blockIdx.x;
  const uint32_t t0 = a.rank_tile0[r], t1 = a.rank_tile0[r + 1];
  const uint32_t tid = threadIdx.x;
  for (int i = tid; i < HASH; i += RS_NT) hset[i] = NONE32;
  if (tid == 0) { nk = 0; npeer = 0; }
  __syncthreads();
  // 1. union of keys
  for (uint32_t t = t0 + tid; t < t1; t += RS_NT) {
    const uint32_t n = a.t_nkeys[t];
    for (uint32_t q = 0; q < n; ++q) {
      const uint32_t key = a.t_keys[(uint64_t)t * KCAP + q];
      uint32_t h = (key * 2654435761u) & (HASH - 1);
      for (;;) {
        const uint32_t old = atomicCAS(&hset[h], NONE32, key);
        if (old == NONE32) { uint32_t i = atomicAdd(&nk, 1u); if (i < RCAP) skeys[i] = key; break; }
        if (old == key) break;
        h = (h + 1) & (HASH - 1);
      }
    }
  }
  __syncthreads();
  const uint32_t C = nk;
  if (C > RCAP) { if (tid == 0) atomicOr(&a.cnt->overflow, 2u); return; }
  // 2. bitonic sort of the rank's keys (ascending = channel order)
  for (int i = tid; i < RCAP; i += RS_NT) if (i >= (int)C) skeys[i] = NONE32;
  __syncthreads();
  for (int k = 2; k <= RCAP; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < RCAP; i += RS_NT) {
        int ixj = i ^ j;
        if (ixj > i) {
          uint32_t x = skeys[i], y = skeys[ixj];
          bool up = (i & k) == 0;
          if ((x > y) == up) { skeys[i] = y; skeys[ixj] = x; }
        }
      }
      __syncthreads();
    }
  for (int i = tid; i < RCAP; i += RS_NT) scarry[i] = 0;
  __syncthreads();
  // 3. chunked scans over the rank's tiles
  const uint64_t rstart = a.rank_off[r];
  uint32_t carry_c = 0, carry_i = 0;
  int32_t carry_j = -1;
  for (uint32_t cb = t0; cb < t1; cb += RS_NT) {
    const uint32_t t = cb + tid;
    const bool in = t < t1;
    const uint32_t nkt = in ? a.t_nkeys[t] : 0;
    for (uint32_t q = 0; q < 8; ++q) tl_keys[tid * 8 + q] = (in && q < nkt) ? a.t_keys[(uint64_t)t * KCAP + q] : NONE32;
    __syncthreads();
    for (uint32_t i = 0; i < C; ++i) {
      const uint32_t key = skeys[i];
      uint32_t v = 0; int pos = -1;
      if (in) {
        for (uint32_t q = 0; q < nkt; ++q) {
          const uint32_t kq = q < 8 ? tl_keys[tid * 8 + q] : a.t_keys[(uint64_t)t * KCAP + q];
          if (kq == key) { pos = (int)q; v = a.t_cnt[(uint64_t)t * KCAP + q]; break; }
        }
      }
      uint32_t tot;
      const uint32_t ex = block_excl_sum<RS_NT>(v, tot, scan_sm);
      if (pos >= 0) a.t_pref[(uint64_t)t * KCAP + pos] = scarry[i] + ex;
      __syncthreads();
      if (tid == 0) scarry[i] += tot;
      __syncthreads();
    }
    const uint32_t nc = in ? a.t_ncomm[t] : 0, ni = in ? a.t_niter[t] : 0;
    uint32_t totc, toti;
    const uint32_t exc = block_excl_sum<RS_NT>(nc, totc, scan_sm) + carry_c;
    const uint32_t exi = block_excl_sum<RS_NT>(ni, toti, scan_sm) + carry_i;
    int32_t lastj = -1;
    if (in) {
      const int32_t lo = a.t_last[t];
      const uint64_t local_start = a.tile_start[t] - rstart;
      if (lo >= 0) lastj = (int32_t)(local_start + (uint64_t)lo - (exc + nc - 1));
    }
    int32_t totj;
    const int32_t exj = block_excl_max<RS_NT>(lastj, totj, scan_smi);
    if (in) {
      a.t_commpre[t] = exc;
      a.t_iterpre[t] = exi;
      a.t_prevj[t] = (uint32_t)max(0, max(carry_j, exj));
    }
    carry_c += totc; carry_i += toti; carry_j = max(carry_j, totj);
    __syncthreads();
  }
  // 4. per-rank outputs
  const uint64_t nr = a.rank_off[r + 1] - rstart;
  for (uint32_t i = tid; i < C; i += RS_NT) {
    a.r_keys[(uint64_t)r * RCAP + i] = skeys[i];
    a.r_cnt[(uint64_t)r * RCAP + i] = scarry[i];
  }
  if (tid == 0) {
    a.r_nkeys[r] = C; a.r_ncomm[r] = carry_c; a.r_niter[r] = carry_i;
    const uint32_t ncomp = (uint32_t)(nr - carry_c);
    a.r_ncomp[r] = ncomp;
    atomicAdd(&a.cnt->n_comm, (unsigned long long)carry_c);
    atomicAdd(&a.cnt->n_comp, (unsigned long long)ncomp);
    atomicMax(&a.cnt->max_niter, carry_i);
    atomicMax(&a.cnt->max_ncomp, ncomp);
    if (nr > 0) {
      const uint32_t last_it = carry_i - ((a.kind[a.rank_off[r + 1] - 1] & 8u) ? 1u : 0u);
      atomicMax(&a.cnt->n_iters, last_it + 1);
    }
  }
  // 5. communicator count extremes (every member contributes, absent = 0) and P2P channels
  for (uint32_t q = a.rcomm_off[r] + tid; q < a.rcomm_off[r + 1]; q += RS_NT) {
    const uint32_t cid = a.rcomm[q];
    uint32_t p = lower_bound_u32(skeys, C, cid);
    const uint32_t v = (p < C && skeys[p] == cid) ? scarry[p] : 0;
    atomicMax(&a.ch_nmax[cid], v);
    atomicMin(&a.ch_nmin[cid], v);
  }
  for (uint32_t i = tid; i < C; i += RS_NT) {
    const uint32_t key = skeys[i];
    if (key < a.n_comms) continue;
    const uint32_t x = key - a.n_comms;
    atomicOr(&a.bitmap[x >> 5], 1u << (x & 31));
    const uint32_t src = x / (uint32_t)a.W, dst = x % (uint32_t)a.W;
    const uint32_t peer = src == r ? dst : src;
    const uint32_t slot = atomicAdd(&npeer, 1u);
    if (slot < PCAP * 2) speer[slot] = peer;
  }
  __syncthreads();
  if (tid == 0) {
    // sort + unique the (few) P2P peers
    uint32_t n = min(npeer, (uint32_t)PCAP * 2);
    for (uint32_t i = 1; i < n; ++i) {
      uint32_t x = speer[i]; int j = (int)i - 1;
      while (j >= 0 && speer[j] > x) { speer[j + 1] = speer[j]; --j; }
      speer[j + 1] = x;
    }
    uint32_t u = 0;
    for (uint32_t i = 0; i < n; ++i) if (u == 0 || speer[u - 1] != speer[i]) speer[u++] = speer[i];
    if (u > PCAP || npeer > PCAP * 2) atomicOr(&a.cnt->overflow, 4u);
    u = min(u, (uint32_t)PCAP);
    for (uint32_t i = 0; i < u; ++i) a.nbp[(uint64_t)r * PCAP + i] = speer[i];
    a.nbp_n[r] = u;
  }
}

int launch_rank_scan(Ctx& c) {
  RankArgs a{c.rank_tile0.as<uint32_t>(), c.rank_off.as<uint64_t>(), c.tile_start.as<uint64_t>(),
             c.t_nkeys.as<uint32_t>(), c.t_keys.as<uint32_t>(), c.t_cnt.as<uint32_t>(), c.t_pref.as<uint32_t>(),
             c.t_ncomm.as<uint32_t>(), c.t_niter.as<uint32_t>(), c.t_last.as<int32_t>(),
             c.t_commpre.as<uint32_t>(), c.t_iterpre.as<uint32_t>(), c.t_prevj.as<uint32_t>(),
             c.r_nkeys.as<uint32_t>(), c.r_keys.as<uint32_t>(), c.r_cnt.as<uint32_t>(), c.r_ncomm.as<uint32_t>(),
             c.r_niter.as<uint32_t>(), c.r_ncomp.as<uint32_t>(),
             c.rcomm_off.as<uint32_t>(), c.rcomm.as<uint32_t>(),
             c.ch_nmax.as<uint32_t>(), c.ch_nmin.as<uint32_t>(), c.bitmap.as<uint32_t>(),
             c.nbp.as<uint32_t>(), c.nbp_n.as<uint32_t>(), c.d_kind, c.W, c.n_comms, c.counters.as<Counters>()};
  k_rank_scan<<<c.W, RS_NT, 0, c.stream>>>(a);
  return 1;
}

// ----------------------------------------------------------------------------- rank prefixes
// Single CTA: exclusive prefixes over ranks (comm / compute / slow-bit-word offsets) and over the
// P2P bitmap words (compact channel ids = popcount prefix, ascending (src,dst)).
constexpr int RP_NT = 1024;
__global__ void __launch_bounds__(RP_NT) k_rank_prefix(int W, const uint32_t* r_ncomm, const uint32_t* r_ncomp,
                                                       uint64_t* r_comm_off, uint64_t* r_comp_off, uint64_t* r_bits_off,
                                                       const uint32_t* bitmap, uint32_t* bitpre, uint64_t n_words,
                                                       Counters* cnt) {
  __shared__ uint32_t sm[33];
  __shared__ unsigned long long carry[3];
  if (threadIdx.x == 0) { carry[0] = carry[1] = carry[2] = 0; }
  __syncthreads();
  for (int b = 0; b < W; b += RP_NT) {
    const int r = b + threadIdx.x;
    const bool in = r < W;
    uint32_t vc = in ? r_ncomm[r] : 0, vp = in ? r_ncomp[r] : 0, vb = in ? (r_ncomp[r] + 31) / 32 : 0;
    uint32_t tc, tp, tb;
    uint32_t ec = block_excl_sum<RP_NT>(vc, tc, sm);
    uint32_t ep = block_excl_sum<RP_NT>(vp, tp, sm);
    uint32_t eb = block_excl_sum<RP_NT>(vb, tb, sm);
    if (in) { r_comm_off[r] = carry[0] + ec; r_comp_off[r] = carry[1] + ep; r_bits_off[r] = carry[2] + eb; }
    __syncthreads();
    if (threadIdx.x == 0) { carry[0] += tc; carry[1] += tp; carry[2] += tb; }
    __syncthreads();
  }
  if (threadIdx.x == 0) { r_comm_off[W] = carry[0]; r_comp_off[W] = carry[1]; r_bits_off[W] = carry[2]; cnt->n_bits_words = carry[2]; }
}

// P2P channel ids = popcount prefix of the W^2-bit bitmap, as a three-kernel multi-CTA scan
// (the bitmap has W^2/32 words: 295K at W = 3072): block sums, one scan of the sums, block scans
constexpr int BP_NT = 1024;
__global__ void __launch_bounds__(BP_NT) k_bitmap_sums(const uint32_t* bitmap, uint64_t n_words, uint32_t* bsum) {
  __shared__ uint32_t sm[33];
  const uint64_t w = (uint64_t)blockIdx.x * BP_NT + threadIdx.x;
  uint32_t tot;
  block_excl_sum<BP_NT>(w < n_words ? (uint32_t)__popc(bitmap[w]) : 0u, tot, sm);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(BP_NT) k_bitmap_scan(uint32_t* bsum, uint32_t nb, Counters* cnt) {
  __shared__ uint32_t sm[33];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t b = 0; b < nb; b += BP_NT) {
    const uint32_t i = b + threadIdx.x;
    const uint32_t v = i < nb ? bsum[i] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_sum<BP_NT>(v, tot, sm);
    if (i < nb) bsum[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) cnt->n_p2p = carry;
}

__global__ void __launch_bounds__(BP_NT) k_bitmap_pre(const uint32_t* bitmap, uint64_t n_words, const uint32_t* bsum, uint32_t* bitpre) {
  __shared__ uint32_t sm[33];
  const uint64_t w = (uint64_t)blockIdx.x * BP_NT + threadIdx.x;
  uint32_t tot;
  const uint32_t ex = block_excl_sum<BP_NT>(w < n_words ? (uint32_t)__popc(bitmap[w]) : 0u, tot, sm);
  if (w < n_words) bitpre[w] = bsum[blockIdx.x] + ex;
}

int launch_rank_prefix(Ctx& c) {
  k_rank_prefix<<<1, RP_NT, 0, c.stream>>>(c.W, c.r_ncomm.as<uint32_t>(), c.r_ncomp.as<uint32_t>(),
                                           c.r_comm_off.as<uint64_t>(), c.r_comp_off.as<uint64_t>(),
                                           c.r_bits_off.as<uint64_t>(), c.bitmap.as<uint32_t>(), c.bitpre.as<uint32_t>(),
                                           c.n_bm_words, c.counters.as<Counters>());
  const uint32_t nb = (uint32_t)((c.n_bm_words + BP_NT - 1) / BP_NT);
  if (c.bmsum.ensure((uint64_t)std::max<uint32_t>(nb, 1) * 4) != cudaSuccess) return 1;
  k_bitmap_sums<<<std::max<uint32_t>(nb, 1), BP_NT, 0, c.stream>>>(c.bitmap.as<uint32_t>(), c.n_bm_words, c.bmsum.as<uint32_t>());
  k_bitmap_scan<<<1, BP_NT, 0, c.stream>>>(c.bmsum.as<uint32_t>(), nb, c.counters.as<Counters>());
  k_bitmap_pre<<<std::max<uint32_t>(nb, 1), BP_NT, 0, c.stream>>>(c.bitmap.as<uint32_t>(), c.n_bm_words, c.bmsum.as<uint32_t>(),
                                                                  c.bitpre.as<uint32_t>());
  return 4;
}

// ----------------------------------------------------------------------------- P2P channels
__device__ __forceinline__ uint32_t p2p_id(const uint32_t* bitmap, const uint32_t* bitpre, uint32_t x) {
  return bitpre[x >> 5] + __popc(bitmap[x >> 5] & ((1u << (x & 31)) - 1u));
}

__global__ void k_p2p_counts(int W, uint32_t n_comms, const uint32_t* r_nkeys, const uint32_t* r_keys,
                             const uint32_t* r_cnt, const uint32_t* bitmap, const uint32_t* bitpre,
                             uint32_t* nsend, uint32_t* nrecv, uint32_t* psrc, uint32_t* pdst) {
  const uint32_t r = blockIdx.x;
  const uint32_t C = r_nkeys[r];
  for (uint32_t i = threadIdx.x; i < C; i += blockDim.x) {
    const uint32_t key = r_keys[(uint64_t)r * RCAP + i];
    if (key < n_comms) continue;
    const uint32_t x = key - n_comms;
    const uint32_t pid = p2p_id(bitmap, bitpre, x);
    const uint32_t src = x / (uint32_t)W, dst = x % (uint32_t)W;
    const uint32_t v = r_cnt[(uint64_t)r * RCAP + i];
    if (src == r) { nsend[pid] = v; psrc[pid] = src; pdst[pid] = dst; }
    else { nrecv[pid] = v; psrc[pid] = src; pdst[pid] = dst; }
  }
}

// Single CTA: per-channel max/min member counts, instance bases and slot bases (exclusive scans).
__global__ void __launch_bounds__(RP_NT) k_channels(uint32_t n_comms, uint64_t NCH, const uint64_t* coff,
                                                    uint32_t* nmax, uint32_t* nmin, const uint32_t* nsend,
                                                    const uint32_t* nrecv, uint64_t* base, uint64_t* slot,
                                                    Counters* cnt) {
  __shared__ unsigned long long sm_w[32];
  __shared__ unsigned long long sm_w2[32];
  __shared__ unsigned long long carry[2];
  if (threadIdx.x == 0) { carry[0] = carry[1] = 0; }
  __syncthreads();
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
  for (uint64_t b = 0; b < NCH; b += RP_NT) {
    const uint64_t ch = b + threadIdx.x;
    unsigned long long v = 0, vs = 0;
    if (ch < NCH) {
      uint32_t mx, mn, nm;
      if (ch < n_comms) {
        nm = (uint32_t)(coff[ch + 1] - coff[ch]);
        mx = nmax[ch]; mn = nm ? nmin[ch] : 0;
      } else {
        const uint64_t p = ch - n_comms;
        mx = max(nsend[p], nrecv[p]); mn = min(nsend[p], nrecv[p]); nm = 2;
      }
      nmax[ch] = mx; nmin[ch] = mn;
      v = mx; vs = (unsigned long long)mx * nm;
    }
    // 64-bit block exclusive scans
    unsigned long long inc = v, incs = vs;
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, inc, o), ts = __shfl_up_sync(0xFFFFFFFFu, incs, o);
      if (lane >= (uint32_t)o) { inc += t; incs += ts; }
    }
    if (lane == 31) { sm_w[wid] = inc; sm_w2[wid] = incs; }
    __syncthreads();
    if (wid == 0) {
      unsigned long long x = sm_w[lane], xs = sm_w2[lane];
      unsigned long long xi = x, xis = xs;
      for (int o = 1; o < 32; o <<= 1) {
        unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, xi, o), ts = __shfl_up_sync(0xFFFFFFFFu, xis, o);
        if (lane >= (uint32_t)o) { xi += t; xis += ts; }
      }
      sm_w[lane] = xi - x; sm_w2[lane] = xis - xs;
      if (lane == 31) { sm_w[31] = xi - x; }
    }
    __syncthreads();
    if (ch < NCH) { base[ch] = carry[0] + sm_w[wid] + inc - v; slot[ch] = carry[1] + sm_w2[wid] + incs - vs; }
    __syncthreads();
    if (threadIdx.x == RP_NT - 1) { carry[0] += sm_w[wid] + inc; carry[1] += sm_w2[wid] + incs; }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    base[NCH] = carry[0]; slot[NCH] = carry[1];
    cnt->n_instances = carry[0]; cnt->n_slots = carry[1];
  }
}

__global__ void k_channel_tail(uint32_t n_comms, const uint64_t* base, const uint64_t* slot, Counters* cnt) {
  cnt->p2p_inst0 = base[n_comms];
  cnt->p2p_slot0 = slot[n_comms];
}

// Index of the cross-stage instances (every channel except TP-/DP-class communicators): exclusive
// scan of their instance counts, so k_cross_reduce runs over exactly those instances.
__global__ void __launch_bounds__(RP_NT) k_cross_index(uint32_t n_comms, uint64_t NCH, const uint8_t* ccls,
                                                       const uint32_t* nmax, uint64_t* xbase, Counters* cnt) {
  __shared__ unsigned long long sm[32];
  __shared__ unsigned long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
  for (uint64_t b = 0; b < NCH; b += RP_NT) {
    const uint64_t ch = b + threadIdx.x;
    unsigned long long v = 0;
    if (ch < NCH) v = (ch >= n_comms || (ccls[ch] != 1 && ccls[ch] != 2)) ? nmax[ch] : 0;
    unsigned long long inc = v;
    for (int o = 1; o < 32; o <<= 1) { unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, inc, o); if (lane >= (uint32_t)o) inc += t; }
    if (lane == 31) sm[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      unsigned long long x = sm[lane], xi = x;
      for (int o = 1; o < 32; o <<= 1) { unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, xi, o); if (lane >= (uint32_t)o) xi += t; }
      sm[lane] = xi - x;
    }
    __syncthreads();
    if (ch < NCH) xbase[ch] = carry + sm[wid] + inc - v;
    __syncthreads();
    if (threadIdx.x == RP_NT - 1) carry += sm[wid] + inc;
    __syncthreads();
  }
  if (threadIdx.x == 0) { xbase[NCH] = carry; cnt->n_xinst = carry; }
}

// P2P member counts only (the shard path builds the channel tables on the host after its exchange)
int launch_p2p_counts_to(Ctx& c, uint32_t* nsend, uint32_t* nrecv, uint32_t* psrc, uint32_t* pdst) {
  k_p2p_counts<<<c.W, 64, 0, c.stream>>>(c.W, c.n_comms, c.r_nkeys.as<uint32_t>(), c.r_keys.as<uint32_t>(),
                                          c.r_cnt.as<uint32_t>(), c.bitmap.as<uint32_t>(), c.bitpre.as<uint32_t>(),
                                          nsend, nrecv, psrc, pdst);
  return 1;
}

int launch_p2p_counts(Ctx& c) {
  if (!c.n_p2p) return 0;
  return launch_p2p_counts_to(c, c.ch_nsend.as<uint32_t>(), c.ch_nrecv.as<uint32_t>(), c.ch_nsend.as<uint32_t>() + c.n_p2p,
                              c.ch_nrecv.as<uint32_t>() + c.n_p2p);
}

int launch_p2p_channels(Ctx& c) {
  int n = 0;
  if (c.n_p2p) {
    k_p2p_counts<<<c.W, 64, 0, c.stream>>>(c.W, c.n_comms, c.r_nkeys.as<uint32_t>(), c.r_keys.as<uint32_t>(),
                                            c.r_cnt.as<uint32_t>(), c.bitmap.as<uint32_t>(), c.bitpre.as<uint32_t>(),
                                            c.ch_nsend.as<uint32_t>(), c.ch_nrecv.as<uint32_t>(),
                                            c.ch_nsend.as<uint32_t>() + c.n_p2p, c.ch_nrecv.as<uint32_t>() + c.n_p2p);
    ++n;
  }
  k_channels<<<1, RP_NT, 0, c.stream>>>(c.n_comms, c.NCH, c.coff.as<uint64_t>(), c.ch_nmax.as<uint32_t>(),
                                        c.ch_nmin.as<uint32_t>(), c.ch_nsend.as<uint32_t>(), c.ch_nrecv.as<uint32_t>(),
                                        c.ch_base.as<uint64_t>(), c.ch_slot.as<uint64_t>(), c.counters.as<Counters>());
  k_channel_tail<<<1, 1, 0, c.stream>>>(c.n_comms, c.ch_base.as<uint64_t>(), c.ch_slot.as<uint64_t>(), c.counters.as<Counters>());
  k_cross_index<<<1, RP_NT, 0, c.stream>>>(c.n_comms, c.NCH, c.ccls.as<uint8_t>(), c.ch_nmax.as<uint32_t>(),
                                           c.xbase.as<uint64_t>(), c.counters.as<Counters>());
  return n + 3;
}

// ----------------------------------------------------------------------------- K1c assign
// Second walk of every warp tile: occurrence index k per event (tile prefix + ordered in-tile
// rank), instance id base(channel)+k, scatter of the member duration / kind into its slot,
// compaction of compute events per rank, per-rank iteration boundaries in compute-index space.
struct AssignArgs {
  TileArgs t;
  const uint32_t* t_nkeys; const uint32_t* t_keys; const uint32_t* t_pref;
  const uint32_t* t_commpre; const uint32_t* t_iterpre;
  const uint64_t* r_comm_off; const uint64_t* r_comp_off;
  const uint32_t* bitmap; const uint32_t* bitpre;
  const uint64_t* ch_base; const uint64_t* ch_slot;
  uint32_t* inst_c; uint4* slots;
  uint32_t* cdur; uint16_t* cop; uint32_t* citer; uint32_t NIT1;
  uint64_t p2p_slot0, p2p_inst0;
};

#ifndef MS_ASSIGN_MINB
#define MS_ASSIGN_MINB 4  // 4 CTAs per SM (64 registers, a few spills): 14.1 -> 11.5 ms on C3's general path
#endif
__global__ void __launch_bounds__(256, MS_ASSIGN_MINB) k_assign(AssignArgs A) {
  __shared__ uint32_t cdb[8][256];  // per warp: the round's compute durations / op ids, compacted
  __shared__ uint16_t cob[8][256];
  const TileArgs& a = A.t;
  const uint32_t wid = threadIdx.x >> 5;
  uint64_t tile = (uint64_t)blockIdx.x * (blockDim.x >> 5) + wid;
  if (tile >= a.n_tiles) return;
  if (a.order) tile = a.order[tile];
  const uint32_t lane = lane_id();
  const uint32_t r = a.tile_rank[tile];
  const uint64_t rstart = a.rank_off[r];
  const uint64_t s = a.tile_start[tile];
  const uint64_t e = min(s + (uint64_t)TILE_EV, a.rank_off[r + 1]);
  // per-lane channel table
  const uint32_t nkeys = A.t_nkeys[tile];
  uint32_t tkey = NONE32, trun = 0, tnmem = 0, tslot = 0, tisp = 0;
  uint64_t tbase = 0, tsbase = 0;
  if (lane < nkeys) {
    tkey = A.t_keys[tile * KCAP + lane];
    trun = A.t_pref[tile * KCAP + lane];
    uint64_t ch;
    if (tkey < a.n_comms) {
      ch = tkey;
      const uint64_t cb = a.coff[tkey];
      tnmem = (uint32_t)(a.coff[tkey + 1] - cb);
      tslot = lower_bound_u32(a.cmem + cb, tnmem, r);
    } else {
      const uint32_t x = tkey - a.n_comms;
      ch = a.n_comms + p2p_id(A.bitmap, A.bitpre, x);
      tnmem = 2; tisp = 1;
      tslot = (x / (uint32_t)a.W == r) ? 0 : 1;
    }
    tbase = A.ch_base[ch]; tsbase = A.ch_slot[ch];
  }
  uint32_t comm_carry = A.t_commpre[tile], iter_carry = A.t_iterpre[tile];
  const uint64_t comm_off = A.r_comm_off[r], comp_off = A.r_comp_off[r];
  uint32_t* citer_r = A.citer + (uint64_t)r * A.NIT1;
  for (uint64_t base = s & ~7ull; base < e; base += 256) {
    const uint64_t g = base + 8ull * lane;
    uint16_t ko[8]; uint32_t cm[8], du[8];
    load8_u16(a.kind, g, a.N, ko);
    load8_u32(a.comm, g, a.N, cm);
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
    // the P2P events' payload / meta words are gathered below: request them now (L2 prefetch)
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (((commm >> q) & 1u) && (ko[q] & 7u) >= 5) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.pay + g + q));
        if ((ko[q] & 7u) == 5) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.meta + g + q));
      }
    uint32_t ctot, itot;
    const uint32_t cex = warp_excl_scan(__popc(commm), ctot) + comm_carry;
    const uint32_t iex = warp_excl_scan(__popc(itm), itot) + iter_carry;
    // compute events (compacted through shared memory: the round's compute events are one contiguous
    // range of the rank's compute index, stored coalesced) and iteration boundaries
    const uint64_t ev0 = base > s ? base : s;  // the round's first event
    const uint32_t jbase = (uint32_t)(ev0 - rstart) - comm_carry;
    uint32_t ncomp = __popc(valid & ~commm);
    ncomp = warp_sum_u32(ncomp);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (!((valid >> q) & 1u)) continue;
      const uint64_t ev = g + q;
      const uint32_t cb = cex + __popc(commm & ((1u << q) - 1u));
      const uint32_t j = (uint32_t)(ev - rstart) - cb;
      const bool isc = !((commm >> q) & 1u);
      if (isc) { cdb[wid][j - jbase] = du[q]; cob[wid][j - jbase] = (uint16_t)(ko[q] >> 4); }
      if ((itm >> q) & 1u) {
        const uint32_t ib = iex + __popc(itm & ((1u << q) - 1u));
        citer_r[ib + 1] = j + (isc ? 1u : 0u);
      }
    }
    __syncwarp();
    for (uint32_t i = lane; i < ncomp; i += 32) { A.cdur[comp_off + jbase + i] = cdb[wid][i]; A.cop[comp_off + jbase + i] = cob[wid][i]; }
    __syncwarp();
    // comm events, one pass per distinct key of the round
    uint32_t keys[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      keys[q] = 0;
      if ((commm >> q) & 1u) {
        const uint32_t kind = ko[q] & 7u;
        keys[q] = kind <= 4 ? cm[q] : a.n_comms + (kind == 5 ? r * (uint32_t)a.W + cm[q] : cm[q] * (uint32_t)a.W + r);
      }
    }
    uint32_t pending = commm;
    while (__any_sync(0xFFFFFFFFu, pending != 0)) {
      const uint32_t leader = __ffs(__ballot_sync(0xFFFFFFFFu, pending != 0)) - 1;
      uint32_t mykey = 0;
      const int first = __ffs(pending) - 1;
#pragma unroll
      for (int q = 0; q < 8; ++q) if (q == first) mykey = keys[q];
      const uint32_t kappa = __shfl_sync(0xFFFFFFFFu, mykey, leader);
      uint32_t m = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) if (((pending >> q) & 1u) && keys[q] == kappa) m |= 1u << q;
      pending &= ~m;
      uint32_t tot;
      const uint32_t kex = warp_excl_scan(__popc(m), tot);
      const uint32_t found = __ballot_sync(0xFFFFFFFFu, tkey == kappa);
      const int tl = __ffs(found) - 1;   // tile table always holds every key of its tile
      const uint32_t run = __shfl_sync(0xFFFFFFFFu, trun, tl);
      const uint64_t kb = __shfl_sync(0xFFFFFFFFu, tbase, tl);
      const uint64_t sb = __shfl_sync(0xFFFFFFFFu, tsbase, tl);
      const uint32_t nmem = __shfl_sync(0xFFFFFFFFu, tnmem, tl);
      const uint32_t mslot = __shfl_sync(0xFFFFFFFFu, tslot, tl);
      const uint32_t isp = __shfl_sync(0xFFFFFFFFu, tisp, tl);
      if (lane == (uint32_t)tl) trun += tot;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (!((m >> q) & 1u)) continue;
        const uint64_t ev = g + q;
        const uint32_t k = run + kex + __popc(m & ((1u << q) - 1u));
        const uint64_t inst = kb + k;
        const uint32_t cb = cex + __popc(commm & ((1u << q) - 1u));
        A.inst_c[comm_off + cb] = (uint32_t)inst;
        const uint64_t si = sb + (uint64_t)k * nmem + mslot;
        const uint32_t kind = ko[q] & 7u;
        const uint32_t warm = kind == 5 ? (a.meta[ev] >> 14) & 1u : 0u;
        A.slots[si] = make_uint4(du[q], 0u, slot_z(iex + __popc(itm & ((1u << q) - 1u)), kind, warm), isp ? a.pay[ev] : 0u);
      }
    }
    comm_carry += ctot;
    iter_carry += itot;
  }
}

int launch_assign(Ctx& c) {
  if (c.n_tiles == 0) return 0;
  AssignArgs A;
  A.t = TileArgs{c.tile_rank.as<uint32_t>(), c.tile_start.as<uint64_t>(), c.rank_off.as<uint64_t>(), c.d_kind, c.d_comm,
                 c.d_dur, c.d_meta, c.d_pay, c.N, c.n_tiles, c.W, c.n_comms, c.coff.as<uint64_t>(), c.cmem.as<uint32_t>(),
                 c.counters.as<Counters>()};
  A.t_nkeys = c.t_nkeys.as<uint32_t>(); A.t_keys = c.t_keys.as<uint32_t>(); A.t_pref = c.t_pref.as<uint32_t>();
  A.t_commpre = c.t_commpre.as<uint32_t>(); A.t_iterpre = c.t_iterpre.as<uint32_t>();
  A.r_comm_off = c.r_comm_off.as<uint64_t>(); A.r_comp_off = c.r_comp_off.as<uint64_t>();
  A.bitmap = c.bitmap.as<uint32_t>(); A.bitpre = c.bitpre.as<uint32_t>();
  A.ch_base = c.ch_base.as<uint64_t>(); A.ch_slot = c.ch_slot.as<uint64_t>();
  A.t.order = tile_order_ptr(c);
  A.inst_c = c.inst_c.as<uint32_t>(); A.slots = c.slots.as<uint4>();
  A.cdur = c.cdur.as<uint32_t>(); A.cop = c.cop.as<uint16_t>(); A.citer = c.citer.as<uint32_t>(); A.NIT1 = c.NIT + 1;
  A.p2p_slot0 = c.p2p_slot0; A.p2p_inst0 = c.p2p_inst0;
  unsigned blocks = (unsigned)((c.n_tiles + 7) / 8);
  k_assign<<<blocks, 256, 0, c.stream>>>(A);
  return 1;
}

// ----------------------------------------------------------------------------- K2 instance reduce
// Per instance: completeness, kind / payload integrity, dmin, dmax, last arriver (lowest slot
// with dur == dmin, reading R20), uniqueness. Record = {dmin, dmax, last_rank, flags | cls<<8}.
__global__ void __launch_bounds__(256) k_inst_reduce(uint64_t n_inst, uint64_t NCH, uint32_t n_comms,
                                                     const uint64_t* ch_base, const uint64_t* ch_slot,
                                                     const uint32_t* ch_nmin, const uint64_t* coff,
                                                     const uint32_t* cmem, const uint8_t* ccls,
                                                     const uint32_t* nsend, const uint32_t* psrc, const uint32_t* pdst,
                                                     const uint4* slots, uint4* rec, unsigned long long* lk_key,
                                                     uint64_t p2p_inst0, Counters* cnt) {
  uint32_t inc = 0, kmis = 0, pmis = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_inst; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t ch = upper_bound_u64(ch_base, NCH + 1, i) - 1;
    const uint64_t k = i - ch_base[ch];
    const bool isp = ch >= n_comms;
    uint32_t nm, cls = 0;
    if (!isp) { nm = (uint32_t)(coff[ch + 1] - coff[ch]); cls = ccls[ch]; } else nm = 2;
    uint32_t flags = 0;
    const uint64_t sb = ch_slot[ch] + k * nm;
    if (isp && k < nsend[ch - n_comms] && (slots[sb].z >> 31)) flags |= SCAN_F_WARMUP;  // the sender's flag
    uint32_t dmin = 0, dmax = 0, last = NONE32;
    if (k < ch_nmin[ch]) {
      flags |= SCAN_F_COMPLETE;
      bool kind_ok = true, pay_ok = true;
      if (!isp) {
        const uint32_t k0 = slot_kind(slots[sb].z);
        for (uint32_t q = 1; q < nm; ++q) if (slot_kind(slots[sb + q].z) != k0) kind_ok = false;
      } else {
        pay_ok = slots[sb].w == slots[sb + 1].w;
      }
      if (kind_ok) flags |= SCAN_F_KIND_OK; else ++kmis;
      if (pay_ok) flags |= SCAN_F_PAYLOAD_OK; else ++pmis;
      if (kind_ok && pay_ok) {
        flags |= SCAN_F_VALID;
        dmin = NONE32; dmax = 0;
        uint32_t ls = 0, nat = 0;
        for (uint32_t q = 0; q < nm; ++q) {
          const uint32_t d = slots[sb + q].x;
          if (d < dmin) { dmin = d; ls = q; nat = 1; } else if (d == dmin) ++nat;
          dmax = max(dmax, d);
        }
        if (nat == 1) flags |= SCAN_F_UNIQUE_LAST;
        if (!isp) last = cmem[coff[ch] + ls];
        else last = ls == 0 ? psrc[ch - n_comms] : pdst[ch - n_comms];
      }
    } else {
      ++inc;
    }
    rec[i] = make_uint4(dmin, dmax, last, flags | (cls << 8));
    if (isp) lk_key[i - p2p_inst0] = lk_sample_key(flags, dmin, (flags & SCAN_F_VALID) ? slots[sb].w : 0u);
  }
  inc = warp_sum_u32(inc); kmis = warp_sum_u32(kmis); pmis = warp_sum_u32(pmis);
  if (lane_id() == 0) {
    if (inc) atomicAdd(&cnt->n_incomplete, (unsigned long long)inc);
    if (kmis) atomicAdd(&cnt->n_kind_mismatch, (unsigned long long)kmis);
    if (pmis) atomicAdd(&cnt->n_payload_mismatch, (unsigned long long)pmis);
  }
}

int launch_inst_reduce(Ctx& c) {
  if (c.n_inst == 0) return 0;
  unsigned blocks = (unsigned)std::min<uint64_t>((c.n_inst + 255) / 256, 148ull * 16);
  k_inst_reduce<<<blocks, 256, 0, c.stream>>>(c.n_inst, c.NCH, c.n_comms, c.ch_base.as<uint64_t>(), c.ch_slot.as<uint64_t>(),
                                              c.ch_nmin.as<uint32_t>(), c.coff.as<uint64_t>(), c.cmem.as<uint32_t>(),
                                              c.ccls.as<uint8_t>(), c.ch_nsend.as<uint32_t>(), c.ch_nsend.as<uint32_t>() + c.n_p2p,
                                              c.ch_nrecv.as<uint32_t>() + c.n_p2p, c.slots.as<uint4>(), c.inst_rec.as<uint4>(),
                                              c.lk_key.as<unsigned long long>(), c.p2p_inst0, c.counters.as<Counters>());
  return 1;
}

}  // namespace ms
