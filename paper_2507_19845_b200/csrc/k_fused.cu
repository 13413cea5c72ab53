// k_fused.cu — K9: the fused SPMD stage-tile pass (the hot path of scan_analyze).
//
// Inside one pipeline stage every TP x DP rank runs the same op sequence ("ranks playing the
// same role ... execute identical sequences of compute kernels"; Megatron's SPMD loop).
// A CTA owns [T positions] x [all R = TP*DP ranks of one stage]: it streams the tile once from
// HBM into shared memory, verifies every event against the stage's template rank (kind_op and
// the communicator / peer its role implies), and computes in the same pass
//   * A1-A2 occurrence index k (template tile bases + in-tile rank per role) and instance ids,
//   * A3 dmin / dmax / last arriver / waits of every TP- and DP-group instance (all members are
//     in the tile), per-rank sums,
//   * A4 leave-one-out lower medians over the DP peers and the slow bits,
//   * A5 stage-2 joined / late counts (the preceding compute segment is in the tile, except for
//     the first comm position of a tile, which is deferred to k_deferred),
//   * A7 wait-for edge weights.
// Cross-stage instances (model-parallel, embedding, P2P) are scattered to their slots and
// finished by k_cross_reduce. Any verification failure sets a flag and the whole analysis is
// redone by the general path (api.cu), so results never depend on the SPMD assumption.
#include <type_traits>
#include "internal.cuh"

#include <cstdlib>

namespace ms {

enum { TY_COMPUTE = 0, TY_TP = 1, TY_DP = 2, TY_XCOLL = 3, TY_P2P = 4 };

// Role of an event on the template rank of its stage: index of its communicator in the rank's
// sorted communicator list (collectives), 16 + 8*send + (stage delta + 4) for P2P; -1 = none.
__device__ __forceinline__ int role_of(uint32_t kind, uint32_t cm, uint32_t r0, const uint32_t* rc, uint32_t ncr,
                                       uint32_t R, int W) {
  if (kind >= 1 && kind <= 4) {
    const uint32_t p = lower_bound_u32(rc, ncr, cm);
    return (p < ncr && rc[p] == cm) ? (int)p : -1;
  }
  if (kind == 5 || kind == 6) {
    if (cm >= (uint32_t)W || cm == r0) return -1;
    const int d = (int)cm - (int)r0;
    if (d % (int)R) return -1;
    const int ds = d / (int)R;
    if (ds == 0 || ds > 3 || ds < -3) return -1;
    return 16 + (kind == 5 ? 8 : 0) + (ds + 4);
  }
  return -1;
}

// ----------------------------------------------------------------------------- F0 pre-pass
// One warp per fused tile reads the template rank's row only (1/R of the data) and derives
// everything the fused kernel needs per position, relative to the tile: role and type, compute /
// comm / iteration index, occurrence index k within the role, compute index of the previous comm
// position. Also the per-tile column totals that k_fused_scan turns into tile bases.
// Packed position words (10-bit fields; positions per tile <= 1024):
//   posA = j_rel | m_rel << 10 | jprev_rel << 20 | first_comm << 30 | iter_end << 31
//   posB = it_rel | k_rel << 10 | role << 20 | type << 25
struct PreArgs {
  const uint16_t* kind; const uint32_t* comm; const uint64_t* rank_off; int W, PP;
  uint32_t T, R, n_ftiles; const uint32_t* st_tile0; const uint32_t* st_npos;
  const uint32_t* role_comm; const uint32_t* ncroles; const uint8_t* role_type;
  uint32_t* cols; uint32_t* posA; uint32_t* posB; uint16_t* posK; Counters* cnt;
  const uint8_t* tile_stage;
};

__global__ void __launch_bounds__(256) k_fused_prepass(PreArgs a) {
  __shared__ uint32_t rcnt[8][ROLES];
  __shared__ uint32_t rcs[8][CROLES];
  const uint32_t wid = threadIdx.x >> 5, lane = lane_id();
  const uint32_t tile = blockIdx.x * 8 + wid;
  rcnt[wid][lane] = 0;
  __syncwarp();
  if (tile >= a.n_ftiles) return;
  const uint32_t s = a.tile_stage[tile];
  const uint32_t p0 = (tile - a.st_tile0[s]) * a.T;
  const uint32_t np = min(a.T, a.st_npos[s] - p0);
  const uint32_t r0 = s * a.R;
  const uint64_t g0 = a.rank_off[r0] + p0;
  const uint32_t ncr = a.ncroles[s];
  if (lane < CROLES) rcs[wid][lane] = a.role_comm[(uint64_t)r0 * CROLES + lane];  // the template's roles, staged
  __syncwarp();
  const uint32_t* rc = rcs[wid];
  // the template row's kind_op / comm words of the whole tile, loaded up front (independent requests)
  constexpr int PC = 4;  // chunks of 32 positions in flight
  uint16_t kpre[PC];
  uint32_t cpre[PC];
  uint32_t cj = 0, cm = 0, ci = 0;
  int32_t lastj = -1;
  bool bad = false;
  const unsigned lt = (1u << lane) - 1u;
  for (uint32_t base = 0; base < np; base += 32) {
    const uint32_t u = (base >> 5) % PC;
    if (u == 0) {
#pragma unroll
      for (int v = 0; v < PC; ++v) {
        const uint32_t pv = base + 32u * v + lane;
        kpre[v] = pv < np ? a.kind[g0 + pv] : (uint16_t)0;
        cpre[v] = pv < np ? a.comm[g0 + pv] : 0u;
      }
    }
    uint16_t ko = 0;
    uint32_t cmw = 0;
#pragma unroll
    for (int v = 0; v < PC; ++v) if ((uint32_t)v == u) { ko = kpre[v]; cmw = cpre[v]; }
    const uint32_t p = base + lane;
    const bool in = p < np;
    const uint32_t kind = ko & 7u;
    const bool isc = in && kind == 0, iscomm = in && kind != 0, ie = in && ((ko >> 3) & 1u);
    int role = 31;
    uint32_t type = 0;
    if (iscomm) {
      role = role_of(kind, cmw, r0, rc, ncr, a.R, a.W);
      if (role < 0) { bad = true; role = 0; }
      type = role >= 16 ? 4u : a.role_type[s * ROLES + role];
    }
    const unsigned bc = __ballot_sync(0xFFFFFFFFu, isc), bm = __ballot_sync(0xFFFFFFFFu, iscomm),
                   bi = __ballot_sync(0xFFFFFFFFu, ie);
    const uint32_t jx = cj + __popc(bc & lt), mx = cm + __popc(bm & lt), ix = ci + __popc(bi & lt);
    const unsigned grp = __match_any_sync(0xFFFFFFFFu, iscomm ? (uint32_t)role : 0xFFu) & bm;
    uint32_t kr = 0;
    if (iscomm) kr = rcnt[wid][role] + __popc(grp & lt);
    __syncwarp();
    if (iscomm && lane == (uint32_t)(__ffs(grp) - 1)) rcnt[wid][role] += __popc(grp);
    __syncwarp();
    const int32_t inc = warp_incl_max(iscomm ? (int32_t)jx : -1);
    int32_t ex = __shfl_up_sync(0xFFFFFFFFu, inc, 1);
    if (lane == 0) ex = -1;
    const int32_t prev = max(lastj, ex);
    const uint32_t first = iscomm && prev < 0 ? 1u : 0u;
    if (in) {
      a.posA[(uint64_t)tile * a.T + p] = jx | (mx << 10) | ((uint32_t)max(prev, 0) << 20) | (first << 30) | ((ie ? 1u : 0u) << 31);
      a.posB[(uint64_t)tile * a.T + p] = ix | (kr << 10) | ((uint32_t)role << 20) | (type << 25);
      a.posK[(uint64_t)tile * a.T + p] = ko;
    }
    lastj = max(lastj, __shfl_sync(0xFFFFFFFFu, inc, 31));
    cj += __popc(bc); cm += __popc(bm); ci += __popc(bi);
  }
  if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(&a.cnt->overflow, NOT_SPMD);
  __syncwarp();
  const uint64_t n = a.n_ftiles;
  a.cols[(uint64_t)lane * n + tile] = rcnt[wid][lane];
  if (lane == 0) {
    a.cols[(uint64_t)(ROLES + 0) * n + tile] = cj;
    a.cols[(uint64_t)(ROLES + 1) * n + tile] = cm;
    a.cols[(uint64_t)(ROLES + 2) * n + tile] = ci;
    a.cols[(uint64_t)(ROLES + 3) * n + tile] = lastj >= 0 ? (uint32_t)lastj : NONE32;  // cc_last
  }
}

// F0b: per (stage, column) exclusive scans over the stage's tiles; stage totals. The compute
// column also yields jprev (compute index of the last comm event before the tile).
constexpr int SC_NT = 1024;
// tb (optional): the same bases tile-major, [tile][40] = FCOLS bases, comm count, compute count, stage
// (one 160-byte record per tile, bulk-copied by k_stage)
__global__ void __launch_bounds__(SC_NT) k_fused_scan(uint32_t n_ftiles, const uint32_t* st_tile0, const uint32_t* cols,
                                                      uint32_t* base, uint32_t* st_tot, uint32_t* tb) {
  __shared__ uint32_t sm[33];
  __shared__ int32_t smi[33];
  const uint32_t s = blockIdx.x, col = blockIdx.y;
  const uint32_t t0 = st_tile0[s], t1 = st_tile0[s + 1], nt = t1 - t0;
  const uint64_t n = n_ftiles;
  const uint32_t per = (nt + SC_NT - 1) / SC_NT;
  const uint32_t a0 = t0 + threadIdx.x * per, a1 = min(t1, a0 + per);
  uint32_t loc = 0;
  for (uint32_t t = a0; t < a1; ++t) loc += cols[(uint64_t)col * n + t];
  uint32_t tot;
  uint32_t ex = block_excl_sum<SC_NT>(loc, tot, sm);
  int32_t jl = -1;
  for (uint32_t t = a0; t < a1; ++t) {
    base[(uint64_t)col * n + t] = ex;
    if (tb) {
      tb[(uint64_t)t * 40 + col] = ex;
      if (col == ROLES) { tb[(uint64_t)t * 40 + FCOLS + 1] = cols[(uint64_t)ROLES * n + t]; tb[(uint64_t)t * 40 + FCOLS + 2] = s; }
      if (col == ROLES + 1) tb[(uint64_t)t * 40 + FCOLS] = cols[(uint64_t)(ROLES + 1) * n + t];
    }
    if (col == ROLES) {  // compute column: last comm j of this tile = j0 + cc_last
      const uint32_t cc = cols[(uint64_t)(ROLES + 3) * n + t];
      if (cc != NONE32) jl = max(jl, (int32_t)(ex + cc));
    }
    ex += cols[(uint64_t)col * n + t];
  }
  if (threadIdx.x == 0) st_tot[s * FCOLS + col] = tot;
  if (col == ROLES) {
    // exclusive max-scan of the per-thread "last comm j" -> jprev of each tile
    int32_t totj;
    const int32_t exj = block_excl_max<SC_NT>(jl, totj, smi);
    int32_t run = exj;
    for (uint32_t t = a0; t < a1; ++t) {
      base[(uint64_t)(ROLES + 3) * n + t] = (uint32_t)max(0, run);
      if (tb) tb[(uint64_t)t * 40 + ROLES + 3] = (uint32_t)max(0, run);
      const uint32_t cc = cols[(uint64_t)(ROLES + 3) * n + t];
      if (cc != NONE32) run = max(run, (int32_t)(base[(uint64_t)ROLES * n + t] + cc));
    }
  }
}

int launch_fused_prepass(Ctx& c) {
  PreArgs a{c.d_kind, c.d_comm, c.rank_off.as<uint64_t>(), c.W, c.PP, c.FT, c.FR, c.n_ftiles, c.st_tile0.as<uint32_t>(),
            c.st_npos.as<uint32_t>(), c.role_comm.as<uint32_t>(), c.ncroles.as<uint32_t>(), c.role_type.as<uint8_t>(),
            c.ft_cols.as<uint32_t>(), c.ft_posA.as<uint32_t>(), c.ft_posB.as<uint32_t>(), c.ft_posK.as<uint16_t>(),
            c.counters.as<Counters>(), c.tile_stage.as<uint8_t>()};
  k_fused_prepass<<<(c.n_ftiles + 7) / 8, 256, 0, c.stream>>>(a);
  k_fused_scan<<<dim3(c.PP, ROLES + 3), SC_NT, 0, c.stream>>>(c.n_ftiles, c.st_tile0.as<uint32_t>(), c.ft_cols.as<uint32_t>(),
                                                              c.ft_base.as<uint32_t>(), c.st_tot.as<uint32_t>(),
                                                              c.use_stage ? c.ft_tbase.as<uint32_t>() : nullptr);
  return 2;
}

// ----------------------------------------------------------------------------- census
// Per rank, from its stage's role totals: the rank's sorted channel keys and counts (as the
// general path's k_rank_scan would find them on an SPMD trace), member-count extremes per
// communicator, the P2P channel bitmap and P2P neighbour lists.
struct CensusArgs {
  int W, TP, DP, PP; uint32_t R, n_comms;
  const uint32_t* st_tot; const uint32_t* role_comm; const uint32_t* ncroles;
  const uint32_t* rcomm_off; const uint32_t* rcomm; const uint64_t* rank_off; const uint16_t* kind;
  uint32_t* r_nkeys; uint32_t* r_keys; uint32_t* r_cnt; uint32_t* r_ncomm; uint32_t* r_niter; uint32_t* r_ncomp;
  uint32_t* ch_nmax; uint32_t* ch_nmin; uint32_t* bitmap; uint32_t* nbp; uint32_t* nbp_n; Counters* cnt;
};

__global__ void k_fused_census(CensusArgs a) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (uint32_t)a.W) return;
  const uint32_t s = r / a.R;
  const uint32_t* tot = a.st_tot + s * FCOLS;
  const uint32_t ncr = a.ncroles[s];
  uint32_t keys[ROLES], cnts[ROLES], n = 0;
  uint32_t peers[ROLES], np = 0;
  for (uint32_t ro = 0; ro < ncr; ++ro)
    if (tot[ro]) { keys[n] = a.role_comm[(uint64_t)r * CROLES + ro]; cnts[n] = tot[ro]; ++n; }
  for (uint32_t ro = 16; ro < ROLES; ++ro) {
    if (!tot[ro]) continue;
    const int ds = (int)(ro & 7u) - 4;
    const bool send = (ro >> 3) & 1u;
    const int peer = (int)r + ds * (int)a.R;
    if (peer < 0 || peer >= a.W) { atomicOr(&a.cnt->overflow, NOT_SPMD); continue; }
    const uint32_t src = send ? r : (uint32_t)peer, dst = send ? (uint32_t)peer : r;
    const uint32_t x = src * (uint32_t)a.W + dst;
    keys[n] = a.n_comms + x; cnts[n] = tot[ro]; ++n;
    atomicOr(&a.bitmap[x >> 5], 1u << (x & 31));
    peers[np++] = (uint32_t)peer;
  }
  for (uint32_t i = 1; i < n; ++i) {  // insertion sort by key (<= 32 keys)
    const uint32_t k = keys[i], v = cnts[i];
    int j = (int)i - 1;
    while (j >= 0 && keys[j] > k) { keys[j + 1] = keys[j]; cnts[j + 1] = cnts[j]; --j; }
    keys[j + 1] = k; cnts[j + 1] = v;
  }
  for (uint32_t i = 0; i < n; ++i) { a.r_keys[(uint64_t)r * RCAP + i] = keys[i]; a.r_cnt[(uint64_t)r * RCAP + i] = cnts[i]; }
  a.r_nkeys[r] = n;
  const uint32_t ncomm = tot[ROLES + 1], ncomp = tot[ROLES], niter = tot[ROLES + 2];
  a.r_ncomm[r] = ncomm; a.r_ncomp[r] = ncomp; a.r_niter[r] = niter;
  atomicAdd(&a.cnt->n_comm, (unsigned long long)ncomm);
  atomicAdd(&a.cnt->n_comp, (unsigned long long)ncomp);
  atomicAdd(&a.cnt->n_bits_words, (unsigned long long)((ncomp + 31) / 32));  // k_rank_prefix rewrites the same sum
  atomicMax(&a.cnt->max_niter, niter);
  atomicMin(&a.cnt->min_niter, niter);
  atomicMax(&a.cnt->max_ncomp, ncomp);
  const uint64_t e1 = a.rank_off[r + 1];
  if (e1 > a.rank_off[r]) atomicMax(&a.cnt->n_iters, niter - ((a.kind[e1 - 1] & 8u) ? 1u : 0u) + 1u);
  if (e1 > a.rank_off[r] && (a.kind[e1 - 1] & 8u)) atomicAdd(&a.cnt->n_end_ranks, 1u);
  for (uint32_t q = a.rcomm_off[r]; q < a.rcomm_off[r + 1]; ++q) {
    const uint32_t cid = a.rcomm[q];
    uint32_t v = 0;
    for (uint32_t i = 0; i < n; ++i) if (keys[i] == cid) v = cnts[i];
    atomicMax(&a.ch_nmax[cid], v);
    atomicMin(&a.ch_nmin[cid], v);
  }
  for (uint32_t i = 1; i < np; ++i) {
    const uint32_t x = peers[i];
    int j = (int)i - 1;
    while (j >= 0 && peers[j] > x) { peers[j + 1] = peers[j]; --j; }
    peers[j + 1] = x;
  }
  uint32_t u = 0;
  for (uint32_t i = 0; i < np; ++i) if (u == 0 || peers[u - 1] != peers[i]) peers[u++] = peers[i];
  for (uint32_t i = 0; i < u; ++i) a.nbp[(uint64_t)r * PCAP + i] = peers[i];
  a.nbp_n[r] = u;
}

int launch_fused_census(Ctx& c) {
  CensusArgs a{c.W, c.TP, c.DP, c.PP, c.FR, c.n_comms, c.st_tot.as<uint32_t>(), c.role_comm.as<uint32_t>(),
               c.ncroles.as<uint32_t>(), c.rcomm_off.as<uint32_t>(), c.rcomm.as<uint32_t>(), c.rank_off.as<uint64_t>(),
               c.d_kind, c.r_nkeys.as<uint32_t>(), c.r_keys.as<uint32_t>(), c.r_cnt.as<uint32_t>(), c.r_ncomm.as<uint32_t>(),
               c.r_niter.as<uint32_t>(), c.r_ncomp.as<uint32_t>(), c.ch_nmax.as<uint32_t>(), c.ch_nmin.as<uint32_t>(),
               c.bitmap.as<uint32_t>(), c.nbp.as<uint32_t>(), c.nbp_n.as<uint32_t>(), c.counters.as<Counters>()};
  k_fused_census<<<(c.W + 127) / 128, 128, 0, c.stream>>>(a);
  return 1;
}

// ----------------------------------------------------------------------------- F1 fused tile kernel
// q = x / d by multiply-high with m = ceil(2^32 / d); exact for x < 2^22 and d <= 1024 (x * (m*d - 2^32) < 2^32).
// ceil(2^32 / d) = floor((2^32 - 1) / d) + 1 for d >= 2 (d | 2^32 or not): one 32-bit division, not
// the 64-bit software division every thread of a tile would otherwise run
struct FDiv { uint32_t d, m; };
__host__ __device__ __forceinline__ FDiv fdiv_make(uint32_t d) {
  return FDiv{d, d <= 1 ? 0u : 0xFFFFFFFFu / d + 1u};
}
__device__ __forceinline__ uint32_t fdiv(uint32_t x, FDiv f) { return f.d <= 1 ? x : __umulhi(x, f.m); }

struct FusedArgs {
  const uint32_t* dur; const uint16_t* kind; const uint16_t* meta; const uint32_t* comm; const uint32_t* pay;
  const uint64_t* rank_off; int TP, DP, PP, W; uint32_t n_comms; uint32_t T, R, n_ftiles, G; bool aligned, aligned8;
  const uint32_t* st_tile0; const uint32_t* st_npos; const uint32_t* ft_base; const uint8_t* tile_stage;
  FDiv fTP, fDP, fR, fG, fCH;
  const uint32_t* posA; const uint32_t* posB; const uint16_t* posK;
  const uint32_t* role_comm; const uint32_t* role_slot; const uint32_t* ncroles; uint32_t NCRM;
  const uint32_t* eidx;  // [W][TP+DP] wait-for edge slot of each TP-group / DP-group partner
  const uint64_t* coff;
  const uint64_t* ch_base; const uint64_t* ch_slot; const uint32_t* bitmap; const uint32_t* bitpre;
  const uint64_t* comm_off; const uint64_t* comp_off; const uint64_t* bits_off;
  uint32_t* inst_c; uint32_t* wait_c; uint32_t* bits; uint32_t* cref; uint4* rec;
  uint4* slots; const uint32_t* p2p_rbase;  // SlotRec per member slot; instance base per (rank, P2P role)
  uint64_t p2p_slot0, p2p_inst0;
  uint32_t* citer; uint32_t NIT1;
  const uint64_t* nbc_off; const uint32_t* nbc; const uint32_t* nbp; const uint32_t* nbp_n; uint64_t nnz_tot, nnz_c;
  unsigned long long* ew; unsigned long long* rk_sum; uint32_t* wl_joined; uint32_t* wl_late;
  uint32_t* wd_total; uint32_t* wd_slow;
  uint32_t* dlate; uint32_t* dinfo;
  uint32_t slow_num, slow_den; unsigned long long slow_margin;
  uint32_t wi, classes, mode; unsigned long long late_margin, wait_margin; int want_ref;
  uint32_t it_off;  // global iteration of this shard's first iteration (0 unsharded)
  uint32_t pf_dist, pf_own, pf_p2p, p2p_defer; uint64_t n_events;  // k_fused_t: L2 prefetch of tile + pf_dist (0 = off), of its own tile, of its P2P payload / meta words; column length
  unsigned long long wi_m;  // ceil(2^64 / wi) for wi > 1: window = umulhi64(iteration, wi_m), exact for 32-bit iterations
  Counters* cnt;
  // byte offsets of the transposed kernel's shared-memory arrays (host-computed, fused_t_layout)
  uint32_t o_rcb, o_coffr, o_sinst, o_sbits, o_sedge, o_rcs, o_rsum, o_gsum, o_sjoin, o_slate, o_rslow, o_pa, o_pb, o_vd,
      o_pk, o_lst, o_cl, o_pcode, o_cinf, o_citp;
};

// window of a (global) iteration, R18: floor(it / wi) by a 64-bit reciprocal, m = ceil(2^64 / wi):
// it*m / 2^64 = it/wi + e with 0 <= e < it/2^64 < 2^-32 <= 1/wi, so the floor is exact
__device__ __forceinline__ uint32_t win_of(const FusedArgs& a, uint32_t it) {
  return a.wi == 0 ? 0u : (a.wi == 1 ? it : (uint32_t)__umul64hi((unsigned long long)it, a.wi_m));
}

constexpr int F_NT = 512;

__device__ __forceinline__ void add_edge(const FusedArgs& a, uint32_t r, uint32_t L, uint32_t win, uint32_t wait) {
  const uint64_t nb0 = a.nbc_off[r], nb1 = a.nbc_off[r + 1];
  uint64_t idx;
  const uint32_t pc = lower_bound_u32(a.nbc + nb0, (uint32_t)(nb1 - nb0), L);
  if (pc < nb1 - nb0 && a.nbc[nb0 + pc] == L) idx = nb0 + pc;
  else idx = a.nnz_c + (uint64_t)r * PCAP + lower_bound_u32(a.nbp + (uint64_t)r * PCAP, a.nbp_n[r], L);
  atomicAdd(&a.ew[(uint64_t)win * a.nnz_tot + idx], (unsigned long long)wait);
}

__device__ __forceinline__ bool sbits_any(const uint32_t* sb, uint32_t wb, uint32_t lo, uint32_t hi) {
  if (lo >= hi) return false;
  const uint32_t w0 = lo >> 5, w1 = (hi - 1) >> 5;
  for (uint32_t w = w0; w <= w1; ++w) {
    uint32_t m = sb[w - wb];
    if (w == w0) m &= 0xFFFFFFFFu << (lo & 31);
    if (w == w1) m &= 0xFFFFFFFFu >> (31 - ((hi - 1) & 31));
    if (m) return true;
  }
  return false;
}

// Duration tile in shared memory: row-major [R][T], 16-byte granules XOR-swizzled per row so that
// both TP groups (consecutive rows) and DP groups (rows TP apart) read a column conflict-light.
__device__ __forceinline__ uint32_t sw_idx(uint32_t row, uint32_t p, uint32_t T) {
  const uint32_t sw = (row ^ (row >> 3)) & 7u;
  return row * T + ((((p >> 2) ^ sw)) << 2) + (p & 3u);
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// exact 64-bit accumulation in shared memory with native 32-bit atomics (a 64-bit shared atomicAdd
// compiles to a CAS loop on sm_100a): add to the low word, carry into the high word on wrap-around
__device__ __forceinline__ void add64_lohi(uint32_t* lo, uint32_t* hi, unsigned long long v) {
  const uint32_t vl = (uint32_t)v, vh = (uint32_t)(v >> 32);
  const uint32_t old = atomicAdd(lo, vl);
  const uint32_t carry = (old + vl < old) ? 1u : 0u;
  if (vh + carry) atomicAdd(hi, vh + carry);
}

template <int P>
__global__ void __launch_bounds__(F_NT, 2) k_fused(FusedArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const uint32_t T = a.T, R = a.R, TP = (uint32_t)a.TP, DP = (uint32_t)a.DP, G = a.G;
  const uint32_t SW = T / 32 + 2;
  // ---- shared memory carve-up (see fused_smem_bytes)
  const uint32_t E = TP + DP, NCRM = a.NCRM;
  uint32_t* sd = (uint32_t*)smem_raw;                                   // R x T (swizzled)
  uint32_t* vd = sd + (uint64_t)R * T;                                  // T verification descriptor (16 B aligned)
  unsigned long long* coffr = (unsigned long long*)(vd + T);            // R comm offsets
  unsigned long long* rcb = coffr + R;                                  // R x NCRM channel bases
  unsigned long long* rsum = rcb + (uint64_t)R * NCRM;                  // R x 2: compute durations, waits
  uint32_t* gsum = (uint32_t*)(rsum + 2 * (uint64_t)R);                 // 2 x (DP + TP): lo / hi words
  uint32_t* sedge = gsum + 2 * (DP + TP);                               // 2 x R x (TP+DP): lo / hi words
  uint32_t* rowg = sedge + 2 * (uint64_t)R * E;                         // R: tp-group | dp-group << 16
  uint32_t* sinst = rowg + R;                                           // T x G
  uint32_t* sbits = sinst + (uint64_t)T * G;                            // R x SW
  uint32_t* rcs = sbits + (uint64_t)R * SW;                             // R x NCRM
  uint32_t* pa = rcs + (uint64_t)R * NCRM;                              // T
  uint32_t* pb = pa + T;                                                // T
  uint32_t* sgw = pb + T;                                               // T pslow segment: word lo | word hi << 16
  uint32_t* sgm0 = sgw + T;                                             // T mask of the low word
  uint32_t* sgm1 = sgm0 + T;                                            // T mask of the high word
  uint32_t* sjoin = sgm1 + T;                                           // R
  uint32_t* slate = sjoin + R;                                          // R
  uint32_t* rslow = slate + R;                                          // R: row has a slow bit in this tile
  uint8_t* gmask = (uint8_t*)(rslow + R);                               // T/4 granule masks: compute | in-block << 4
  uint16_t* pk = reinterpret_cast<uint16_t*>(smem_raw + ((((uint8_t*)(gmask + T / 4) - smem_raw) + 15) & ~15));  // 16 B aligned
  uint16_t* lst = pk + T;                                               // 4 x T
  uint16_t* cl = lst + 4 * T;                                           // T: comm positions by m, | class << 14
  __shared__ uint32_t kbase[ROLES];
  __shared__ uint32_t nlist[4];
  __shared__ int32_t dpos;
  __shared__ uint32_t bad, anyslow;

  const uint32_t tile = blockIdx.x;
  const uint32_t tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
  const uint32_t s = a.tile_stage[tile];
  const uint32_t p0 = (tile - a.st_tile0[s]) * T;
  const uint32_t npos = a.st_npos[s];
  const uint32_t np = min(T, npos - p0);
  const uint32_t sbase = s * R;
  const uint64_t n = a.n_ftiles;
  const uint64_t rbase = a.rank_off[sbase];  // SPMD stage: equal counts, rank_off[sbase+row] = rbase + row*npos
  const FDiv fTP = a.fTP, fDP = a.fDP, fR = a.fR;
  const uint32_t ngr = (np + 3) / 4;
  const uint32_t nch = (np + 127) / 128;
  const FDiv fg = ngr == T / 4 ? a.fG : fdiv_make(ngr);
  const FDiv fch = nch == (T + 127) / 128 ? a.fCH : fdiv_make(nch);

  // ---- (1) stream the duration rows of all R ranks into shared memory (async, 16 B granules)
  for (uint32_t i = tid; i < R * ngr; i += F_NT) {
    const uint32_t row = fdiv(i, fg), gi = i - row * ngr;
    const uint64_t g = rbase + (uint64_t)row * npos + p0 + 4 * gi;
    uint32_t* dst = sd + row * T + (((4 * gi) ^ (((row ^ (row >> 3)) & 7u) << 2)));
    if (a.aligned && 4 * gi + 4 <= np) {
      cp_async16(dst, a.dur + g);
    } else {
      for (uint32_t q = 0; q < 4; ++q) dst[q] = 4 * gi + q < np ? a.dur[g + q] : 0u;
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
  // ---- (2) per-tile tables and template position info (from the pre-pass)
  const uint32_t j0 = a.ft_base[(uint64_t)ROLES * n + tile];
  const uint32_t m0 = a.ft_base[(uint64_t)(ROLES + 1) * n + tile];
  const uint32_t it0 = a.ft_base[(uint64_t)(ROLES + 2) * n + tile];  // shard-local iteration (citer index)
  const uint32_t itg0 = it0 + a.it_off;  // global iteration: windows, sit, p2p_iter
  const uint32_t jp0 = a.ft_base[(uint64_t)(ROLES + 3) * n + tile];
  const uint32_t wb = j0 >> 5;
  const uint32_t w_tile = win_of(a, itg0);
  const uint32_t ncr = a.ncroles[s];
  if (tid < ROLES) kbase[tid] = a.ft_base[(uint64_t)tid * n + tile];
  if (tid < 4) nlist[tid] = 0;
  if (tid == 0) { dpos = -1; bad = 0; anyslow = 0; }
  for (uint32_t i = tid; i < R * SW; i += F_NT) sbits[i] = 0;
  for (uint32_t i = tid; i < R; i += F_NT) {
    sjoin[i] = 0; slate[i] = 0; coffr[i] = a.comm_off[sbase + i];
    const uint32_t gt = fdiv(i, fTP);
    rowg[i] = gt | ((i - gt * TP) << 16);
  }
  for (uint32_t i = tid; i < 2 * (DP + TP); i += F_NT) gsum[i] = 0;
  for (uint32_t i = tid; i < 2 * R * E; i += F_NT) sedge[i] = 0;
  for (uint32_t i = tid; i < T / 4; i += F_NT) gmask[i] = 0;
  for (uint32_t i = tid; i < R * ncr; i += F_NT) {
    const uint32_t row = i / ncr, ro = i - row * ncr;
    const uint32_t cid = a.role_comm[(uint64_t)(sbase + row) * CROLES + ro];
    rcs[row * NCRM + ro] = cid;
    rcb[row * NCRM + ro] = a.ch_base[cid];
  }
  for (uint32_t p = tid; p < T; p += F_NT) {
    pa[p] = p < np ? a.posA[(uint64_t)tile * T + p] : 0u;
    pb[p] = p < np ? a.posB[(uint64_t)tile * T + p] : 0u;
    pk[p] = p < np ? a.posK[(uint64_t)tile * T + p] : (uint16_t)0;
  }
  __syncthreads();
  // position lists, comm positions in m order, verification descriptors, pslow segments, granule masks
  for (uint32_t p = tid; p < np; p += F_NT) {
    const uint32_t A = pa[p], B = pb[p];
    const uint32_t ty = (B >> 25) & 7u, role = (B >> 20) & 31u;
    const bool isc = (pk[p] & 7u) == 0;
    const uint32_t li = isc ? 0u : (ty == TY_TP ? 1u : (ty == TY_DP ? 2u : 3u));
    const uint32_t sl = atomicAdd(&nlist[li], 1u);
    lst[li * T + sl] = (uint16_t)p;
    if (isc) {
      vd[p] = 0;
      atomicOr((uint32_t*)(gmask + ((p >> 2) & ~3u)), 1u << (8 * ((p >> 2) & 3u) + (p & 3u)));
    } else {
      cl[(A >> 10) & 1023u] = (uint16_t)(p | ((li - 1u) << 14));
      vd[p] = role < 16 ? (1u | (role << 2)) : (2u | ((uint32_t)(((int)(role & 7u) - 4) * (int)R + 0x100000) << 2));
      if (li < 3) atomicOr((uint32_t*)(gmask + ((p >> 2) & ~3u)), 1u << (8 * ((p >> 2) & 3u) + 4 + (p & 3u)));
      if (((A >> 30) & 1u) && li < 3 && a.mode == 0 && jp0 < j0) dpos = (int32_t)p;
      const uint32_t jp = j0 + (A & 1023u);
      const uint32_t jprev = ((A >> 30) & 1u) ? jp0 : j0 + ((A >> 20) & 1023u);
      if (jprev < jp && jprev >= j0) {
        const uint32_t w0 = jprev >> 5, w1 = (jp - 1) >> 5;
        uint32_t m0_ = 0xFFFFFFFFu << (jprev & 31), m1_ = 0xFFFFFFFFu >> (31 - ((jp - 1) & 31));
        if (w0 == w1) { m0_ &= m1_; m1_ = 0; }
        sgw[p] = (w0 - wb) | ((w1 - wb) << 16);
        sgm0[p] = m0_; sgm1[p] = m1_;   // segments span at most two words when shorter than 33 ops
        if (w1 > w0 + 1) sgm0[p] = 0xFFFFFFFFu, sgm1[p] = 0xFFFFFFFFu, sgw[p] |= 0x80000000u;  // long: slow path
      } else {
        sgw[p] = 0; sgm0[p] = 0; sgm1[p] = 0;
      }
    }
  }
  __syncthreads();
  // ---- (3) verify every rank row's kind_op column against the template, 8 positions per 16-byte
  // load (the comm field is verified in the flush, which visits every comm event anyway)
  {
    const uint32_t n8 = (np + 7) / 8;
    const FDiv f8 = fdiv_make(n8);
    bool mis = false;
    for (uint32_t i = tid; i < R * n8; i += F_NT) {
      const uint32_t row = fdiv(i, f8), g8 = i - row * n8;
      const uint32_t pbase = g8 * 8;
      const uint64_t g = rbase + (uint64_t)row * npos + p0 + pbase;
      const uint4 tv = *reinterpret_cast<const uint4*>(pk + pbase);
      if (a.aligned && pbase + 8 <= np) {
        const uint2 ka = __ldg(reinterpret_cast<const uint2*>(a.kind + g));
        const uint2 kb = __ldg(reinterpret_cast<const uint2*>(a.kind + g + 4));
        mis |= (ka.x != tv.x) | (ka.y != tv.y) | (kb.x != tv.z) | (kb.y != tv.w);
      } else {
        for (uint32_t q = 0; q < 8 && pbase + q < np; ++q) mis |= a.kind[g + q] != pk[pbase + q];
      }
    }
    if (__any_sync(0xFFFFFFFFu, mis) && lane == 0) bad = 1;
  }
  cp_async_wait_all();
  __syncthreads();
  if (bad) { if (tid == 0) atomicOr(&a.cnt->overflow, NOT_SPMD); return; }
  // ---- (4) phase A: stage 1 on every compute position (LOO lower median over the DP peers).
  // Exact quick reject: if den*max <= num*min over the group, no member can be slow (ref >= min).
  const uint32_t nc = nlist[0];
  if (P >= 2) {
    const int q = ((int)DP - 2) / 2;
    const int L = P / 2 - 1 - q;  // low sentinels put s[q], s[q+1] at the fixed indices P/2-1, P/2
    for (uint32_t it = tid; it < nc * TP; it += F_NT) {
      const uint32_t pi = fdiv(it, fTP), tp = it - pi * TP;
      const uint32_t p = lst[pi];
      const uint32_t pq = p & ~3u, pr = p & 3u;
      uint32_t x[P];
      uint32_t mn = 0xFFFFFFFFu, mx = 0;
#pragma unroll
      for (int d = 0; d < P; ++d) {
        const uint32_t row = tp + TP * (uint32_t)d;
        const uint32_t sw4 = ((row ^ (row >> 3)) & 7u) << 2;
        x[d] = d < (int)DP ? sd[row * T + (pq ^ sw4) + pr] : 0u;
        if (d < (int)DP) { mn = min(mn, x[d]); mx = max(mx, x[d]); }
      }
      const bool maybe = (unsigned long long)a.slow_den * mx > (unsigned long long)a.slow_num * mn;
      if (!maybe && !a.want_ref) continue;
      uint32_t v[P];
#pragma unroll
      for (int d = 0; d < P; ++d) v[d] = d < (int)DP ? x[d] : (d < (int)DP + L ? 0u : 0xFFFFFFFFu);
#pragma unroll
      for (int k = 2; k <= P; k <<= 1)
#pragma unroll
        for (int jj = k >> 1; jj > 0; jj >>= 1)
#pragma unroll
          for (int i = 0; i < P; ++i) {
            const int ixj = i ^ jj;
            if (ixj > i) {
              const bool up = (i & k) == 0;
              const uint32_t lo = min(v[i], v[ixj]), hi = max(v[i], v[ixj]);
              v[i] = up ? lo : hi; v[ixj] = up ? hi : lo;
            }
          }
      const uint32_t va = v[P / 2 - 1], vb = v[P / 2];
      const uint32_t j = j0 + (pa[p] & 1023u);
      const uint32_t jw = (j >> 5) - wb, jb = 1u << (j & 31);
#pragma unroll
      for (int d = 0; d < P; ++d) {
        if (d < (int)DP) {
          const uint32_t ref = x[d] > va ? va : vb;
          const unsigned long long du = x[d];
          const bool slow = maybe && (unsigned long long)a.slow_den * du > (unsigned long long)a.slow_num * ref &&
                            du > (unsigned long long)ref + a.slow_margin;
          const uint32_t row = tp + TP * d;
          if (slow) { atomicOr(&sbits[row * SW + jw], jb); anyslow = 1; }
          if (a.want_ref) a.cref[a.comp_off[sbase + row] + j] = ref;
        }
      }
    }
  }
  // iteration boundaries (compute index at which the next iteration starts), every rank
  for (uint32_t p = tid; p < np; p += F_NT) {
    if (!(pa[p] >> 31)) continue;
    const uint32_t v = j0 + (pa[p] & 1023u) + ((pk[p] & 7u) == 0 ? 1u : 0u);
    const uint32_t itp = it0 + (pb[p] & 1023u);
    for (uint32_t row = 0; row < R; ++row) a.citer[(uint64_t)(sbase + row) * a.NIT1 + itp + 1] = v;
  }
  __syncthreads();
  const bool tslow = anyslow != 0;
  if (tslow)
    for (uint32_t row = tid; row < R; row += F_NT) {
      uint32_t o = 0;
      for (uint32_t w = 0; w < SW; ++w) o |= sbits[row * SW + w];
      rslow[row] = o != 0;
    }
  __syncthreads();
  // ---- (5) phase B: TP / DP instances (all members in the tile) and cross-stage scatters
  const uint32_t ntp = nlist[1], ndp = nlist[2], nx = nlist[3];
  const uint32_t I1 = ntp * DP, I2 = I1 + ndp * TP, I3 = I2 + nx * R;
  for (uint32_t it = tid; it < I3; it += F_NT) {
    if (it < I2) {
      const bool istp = it < I1;
      uint32_t p, g;
      if (istp) { const uint32_t pi = fdiv(it, fDP); g = it - pi * DP; p = lst[T + pi]; }
      else { const uint32_t x = it - I1, pi = fdiv(x, fTP); g = x - pi * TP; p = lst[2 * T + pi]; }
      const uint32_t nm = istp ? TP : DP, stride = istp ? 1u : TP, row0 = istp ? TP * g : g;
      const uint32_t B = pb[p];
      const uint32_t role = (B >> 20) & 31u;
      const uint64_t inst = rcb[row0 * NCRM + role] + kbase[role] + ((B >> 10) & 1023u);
      const uint32_t pq = p & ~3u, pr = p & 3u;
      uint32_t dmin = 0xFFFFFFFFu, dmax = 0, ls = 0, nat = 0;
      for (uint32_t q = 0; q < nm; ++q) {
        const uint32_t row = row0 + q * stride;
        const uint32_t d = sd[row * T + (pq ^ (((row ^ (row >> 3)) & 7u) << 2)) + pr];
        if (d < dmin) { dmin = d; ls = q; nat = 1; } else if (d == dmin) ++nat;
        dmax = max(dmax, d);
      }
      const uint32_t cls = istp ? 1u : 2u;
      const uint32_t last = sbase + row0 + ls * stride;
      a.rec[inst] = make_uint4(dmin, dmax, last, (SCAN_F_COMPLETE | SCAN_F_KIND_OK | SCAN_F_PAYLOAD_OK | SCAN_F_VALID |
                                                  (nat == 1 ? SCAN_F_UNIQUE_LAST : 0u)) | (cls << 8));
      sinst[p * G + g] = (uint32_t)inst;
      {
        const uint32_t gi = istp ? g : DP + g;
        add64_lohi(&gsum[gi], &gsum[DP + TP + gi], dmin);
      }
      const uint32_t win = win_of(a, itg0 + (B & 1023u));
      const bool elig = (a.classes >> (cls - 1)) & 1u;
      const bool late_ok = nat == 1 && (unsigned long long)(dmax - dmin) > a.late_margin;
      const uint32_t eslot = istp ? ls : TP + ls;  // partner slot of the last arriver
      const bool isdef = (int32_t)p == dpos;
      const bool chk = elig && (a.mode || tslow || isdef);
      const uint32_t gw = sgw[p], g0 = sgm0[p], g1 = sgm1[p];
      for (uint32_t q = 0; q < nm; ++q) {
        const uint32_t row = row0 + q * stride;
        const uint32_t idx = row * T + (pq ^ (((row ^ (row >> 3)) & 7u) << 2)) + pr;
        const uint32_t wait = sd[idx] - dmin;
        sd[idx] = wait;  // the duration tile now holds the wait at in-block comm positions
        if (q != ls && (unsigned long long)wait > a.wait_margin) {
          if (win == w_tile) add64_lohi(&sedge[row * E + eslot], &sedge[R * E + row * E + eslot], wait);
          else atomicAdd(&a.ew[(uint64_t)win * a.nnz_tot + a.eidx[(uint64_t)(sbase + row) * E + eslot]], (unsigned long long)wait);
        }
        if (!chk) continue;
        const bool lt = q == ls && late_ok;
        if (isdef) {
          if (lt) atomicOr(&a.dlate[(uint64_t)tile * ((R + 31) / 32) + row / 32], 1u << (row & 31));
          continue;
        }
        bool pslow = a.mode != 0;
        if (!pslow && rslow[row]) {
          const uint32_t* sb = sbits + row * SW;
          if (gw & 0x80000000u) {
            const uint32_t jp = j0 + (pa[p] & 1023u);
            pslow = sbits_any(sb, wb, ((pa[p] >> 30) & 1u) ? jp0 : j0 + ((pa[p] >> 20) & 1023u), jp);
          } else {
            pslow = (sb[gw & 0xFFFFu] & g0) | (sb[gw >> 16] & g1);
          }
        }
        if (!pslow) continue;
        if (win == w_tile) { atomicAdd(&sjoin[row], 1u); if (lt) atomicAdd(&slate[row], 1u); }
        else {
          const uint32_t r = sbase + row;
          atomicAdd(&a.wl_joined[(uint64_t)win * a.W + r], 1u);
          if (lt) atomicAdd(&a.wl_late[(uint64_t)win * a.W + r], 1u);
        }
      }
    } else {
      const uint32_t x = it - I2;
      const uint32_t pi = fdiv(x, fR), row = x - pi * R, r = sbase + row;
      const uint32_t p = lst[3 * T + pi];
      const uint32_t A = pa[p], B = pb[p];
      const uint32_t role = (B >> 20) & 31u;
      const uint64_t e = rbase + (uint64_t)row * npos + p0 + p;
      const uint32_t kk = kbase[role] + ((B >> 10) & 1023u);
      uint64_t inst, si;
      uint32_t pay = 0, warm = 0;
      if (role < 16) {
        const uint32_t cid = rcs[row * NCRM + role];
        const uint32_t nm = (uint32_t)(a.coff[cid + 1] - a.coff[cid]);
        inst = a.ch_base[cid] + kk;
        si = a.ch_slot[cid] + (uint64_t)kk * nm + a.role_slot[(uint64_t)r * CROLES + role];
      } else {  // a P2P instance's send / receive slots sit at p2p_slot0 + 2 (inst - p2p_inst0) + 0 / 1
        const bool send = (role >> 3) & 1u;
        const uint32_t rb = a.p2p_rbase[(uint64_t)r * 16 + (role - 16)];
        if (rb == NONE32) { atomicOr(&a.cnt->overflow, NOT_SPMD); continue; }  // no such link: not the template's trace
        inst = (uint64_t)rb + kk;
        si = a.p2p_slot0 + 2 * (inst - a.p2p_inst0) + (send ? 0 : 1);
        pay = a.pay[e];
        if (send) warm = ((uint32_t)a.meta[e] >> 14) & 1u;
      }
      const uint32_t idx = sw_idx(row, p, T);
      const uint32_t itp = itg0 + (B & 1023u);
      a.slots[si] = make_uint4(sd[idx], (uint32_t)(coffr[row] + m0 + ((A >> 10) & 1023u)), slot_z(itp, pk[p], warm), pay);
      sd[idx] = (uint32_t)inst;  // cross positions: the tile now holds the instance id
    }
  }
  __syncthreads();
  // ---- (6) flush: coalesced per-rank inst / wait rows, per-rank sums, slow bits, counters
  const uint32_t ncm = nlist[1] + nlist[2] + nlist[3];
  {
    const FDiv fm = fdiv_make(ncm > 0 ? ncm : 1u);
    bool mis = false;
    for (uint32_t i = tid; i < R * ncm; i += F_NT) {  // consecutive threads: consecutive comm events of a rank
      const uint32_t row = fdiv(i, fm), j = i - row * ncm;
      const uint32_t rg = rowg[row];
      const uint32_t cv = cl[j];
      const uint32_t p = cv & 0x3FFFu, cls = cv >> 14;  // 0 TP, 1 DP, 2 cross
      const uint32_t cm = __ldg(a.comm + rbase + (uint64_t)row * npos + p0 + p);
      // verify the comm field: communicator of the role (collective) or peer of the role (P2P)
      const uint32_t dv = vd[p], t = dv & 3u, x = dv >> 2;
      const uint32_t e1 = rcs[row * NCRM + (t == 1 ? x : 0u)];
      mis |= cm != (t == 1 ? e1 : sbase + row + x - 0x100000u);
      const uint32_t v = sd[row * T + ((p & ~3u) ^ (((row ^ (row >> 3)) & 7u) << 2)) + (p & 3u)];
      const uint32_t si = sinst[cls < 2 ? p * G + (cls == 0 ? (rg & 0xFFFFu) : (rg >> 16)) : 0u];
      uint32_t* dst = a.inst_c + coffr[row] + m0 + j;
      *dst = cls < 2 ? si : v;
      a.wait_c[dst - a.inst_c] = cls < 2 ? v : 0u;  // cross positions: placeholder (k_xwait_scatter), full sectors
    }
    if (__any_sync(0xFFFFFFFFu, mis) && lane == 0) atomicOr(&a.cnt->overflow, NOT_SPMD);
  }
  // per-rank sums: compute durations and waits (the tile now holds waits at in-block comm positions);
  // one thread per row walks its row by 16-byte granules -> no cross-lane reductions
  for (uint32_t row = tid; row < R; row += F_NT) {
    const uint32_t rT = row * T, sw4 = ((row ^ (row >> 3)) & 7u) << 2;
    unsigned long long sc = 0, sw = 0;
    for (uint32_t gi = 0; gi < ngr; ++gi) {
      const uint32_t gm = gmask[gi];
      if (!gm) continue;
      const uint4 v = *reinterpret_cast<const uint4*>(sd + rT + ((4 * gi) ^ sw4));
      const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if ((gm >> q) & 1u) sc += vv[q];
        if ((gm >> (4 + q)) & 1u) sw += vv[q];
      }
    }
    rsum[2 * row] = sc; rsum[2 * row + 1] = sw;
  }
  // stage-1 counters per (window, rank): total = compute positions of the tile, slow = its slow bits
  const uint32_t it_last = itg0 + (np ? (pb[np - 1] & 1023u) : 0u);
  const bool one_window = !a.wi || (win_of(a, itg0) == win_of(a, it_last));
  if (P >= 2 && nc) {
    if (one_window) {
      for (uint32_t row = tid; row < R; row += F_NT) {
        const uint32_t r = sbase + row;
        uint32_t sl = 0;
        if (tslow) for (uint32_t w = 0; w < SW; ++w) sl += __popc(sbits[row * SW + w]);
        atomicAdd(&a.wd_total[(uint64_t)w_tile * a.W + r], nc);
        if (sl) atomicAdd(&a.wd_slow[(uint64_t)w_tile * a.W + r], sl);
      }
    } else {
      for (uint32_t i = tid; i < R * nc; i += F_NT) {
        const uint32_t row = i / nc, p = lst[i - row * nc], r = sbase + row;
        const uint32_t win = win_of(a, itg0 + (pb[p] & 1023u));
        const uint32_t j = j0 + (pa[p] & 1023u);
        atomicAdd(&a.wd_total[(uint64_t)win * a.W + r], 1u);
        if ((sbits[row * SW + (j >> 5) - wb] >> (j & 31)) & 1u) atomicAdd(&a.wd_slow[(uint64_t)win * a.W + r], 1u);
      }
    }
  }
  for (uint32_t row = tid; row < R; row += F_NT) {
    const uint32_t r = sbase + row;
    const uint32_t gt = rowg[row] & 0xFFFFu, gd = rowg[row] >> 16;
    const uint32_t GO = DP + TP;
    const unsigned long long tr = ((unsigned long long)gsum[GO + gt] << 32 | gsum[gt]) +
                                  ((unsigned long long)gsum[GO + DP + gd] << 32 | gsum[DP + gd]);
    if (rsum[2 * row]) atomicAdd(&a.rk_sum[r], rsum[2 * row]);
    if (rsum[2 * row + 1]) atomicAdd(&a.rk_sum[a.W + r], rsum[2 * row + 1]);
    if (tr) atomicAdd(&a.rk_sum[2 * a.W + r], tr);
    if (sjoin[row]) atomicAdd(&a.wl_joined[(uint64_t)w_tile * a.W + r], sjoin[row]);
    if (slate[row]) atomicAdd(&a.wl_late[(uint64_t)w_tile * a.W + r], slate[row]);
  }
  for (uint32_t i = tid; i < R * E; i += F_NT) {
    const unsigned long long v = (unsigned long long)sedge[R * E + i] << 32 | sedge[i];
    if (v) atomicAdd(&a.ew[(uint64_t)w_tile * a.nnz_tot + a.eidx[(uint64_t)sbase * E + i]], v);
  }
  if (nc && tslow) {
    const uint32_t w_first = j0 >> 5, w_last = (j0 + nc - 1) >> 5;
    const uint32_t nw = w_last - w_first + 1;
    for (uint32_t i = tid; i < R * nw; i += F_NT) {
      const uint32_t row = i / nw, w = w_first + (i - row * nw);
      const uint32_t v = sbits[row * SW + (w - wb)];
      if (v) atomicOr(&a.bits[a.bits_off[sbase + row] + w], v);
    }
  }
  if (tid == 0) {
    uint32_t* di = a.dinfo + (uint64_t)tile * 4;
    if (dpos >= 0) {
      const uint32_t p = (uint32_t)dpos;
      const uint32_t ty = (pb[p] >> 25) & 7u;
      di[0] = j0 + (pa[p] & 1023u); di[1] = jp0; di[2] = win_of(a, itg0 + (pb[p] & 1023u)); di[3] = 1u | (ty << 8);
    } else {
      di[3] = 0;
    }
  }
}

// =============================================================================================
// k_fused_t — transposed variant (TP divides 32, R = TP*DP <= 256): the tile is stored position-
// major, sd[p][row] with a padded row of R+1 words, and one warp processes one position at a time:
// lane l owns rows l + 32k. A TP group (TP consecutive rows) sits in TP consecutive lanes of one
// register; a DP group (rows with equal row mod TP) is every lane with equal l mod TP, so both
// reductions are butterflies of shuffles. The load pass transposes in registers and verifies the
// kind_op and comm columns while the data is in registers.
#ifndef MS_FT_NT
#define MS_FT_NT 1024
#endif
#ifndef MS_FT_MINB
#define MS_FT_MINB (1024 / MS_FT_NT)
#endif
constexpr int FT_NT = MS_FT_NT, FT_NW = FT_NT / 32, NRLM = 8, FT_MINB = MS_FT_MINB;  // 32 warps per SM by default

template <int P>
__device__ __forceinline__ void loo_group(const FusedArgs& a, const uint32_t* col, uint32_t tp, uint32_t TP, uint32_t DP, uint32_t j,
                          uint32_t* sbits, uint32_t SW, uint32_t wb, uint32_t sbase, bool& slow_any) {
  const int q = ((int)DP - 2) / 2;
  const int L = P / 2 - 1 - q;
  uint32_t x[P], v[P];
#pragma unroll
  for (int d = 0; d < P; ++d) {
    x[d] = d < (int)DP ? col[tp + TP * d] : 0u;
    v[d] = d < (int)DP ? x[d] : (d < (int)DP + L ? 0u : 0xFFFFFFFFu);
  }
#pragma unroll
  for (int k = 2; k <= P; k <<= 1)
#pragma unroll
    for (int jj = k >> 1; jj > 0; jj >>= 1)
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const int ixj = i ^ jj;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const uint32_t lo = min(v[i], v[ixj]), hi = max(v[i], v[ixj]);
          v[i] = up ? lo : hi; v[ixj] = up ? hi : lo;
        }
      }
  const uint32_t va = v[P / 2 - 1], vb = v[P / 2];
  const uint32_t jw = (j >> 5) - wb, jb = 1u << (j & 31);
#pragma unroll
  for (int d = 0; d < P; ++d) {
    if (d < (int)DP) {
      const uint32_t ref = x[d] > va ? va : vb;
      const unsigned long long du = x[d];
      const bool slow = (unsigned long long)a.slow_den * du > (unsigned long long)a.slow_num * ref &&
                        du > (unsigned long long)ref + a.slow_margin;
      const uint32_t row = tp + TP * d;
      if (slow) { atomicOr(&sbits[row * SW + jw], jb); slow_any = true; }
      if (a.want_ref) a.cref[a.comp_off[sbase + row] + j] = ref;
    }
  }
}

__device__ __forceinline__ void loo_dispatch(const FusedArgs& a, const uint32_t* col, uint32_t tp, uint32_t TP, uint32_t DP,
                                             uint32_t j, uint32_t* sbits, uint32_t SW, uint32_t wb, uint32_t sbase, bool& any) {
  if (DP <= 2) loo_group<2>(a, col, tp, TP, DP, j, sbits, SW, wb, sbase, any);
  else if (DP <= 4) loo_group<4>(a, col, tp, TP, DP, j, sbits, SW, wb, sbase, any);
  else if (DP <= 8) loo_group<8>(a, col, tp, TP, DP, j, sbits, SW, wb, sbase, any);
  else if (DP <= 16) loo_group<16>(a, col, tp, TP, DP, j, sbits, SW, wb, sbase, any);
  else loo_group<32>(a, col, tp, TP, DP, j, sbits, SW, wb, sbase, any);
}

// L2 prefetch of every rank row of fused tile t (dur, comm, kind columns; 128-byte lines, clamped to
// the columns). A hint only.
__device__ __forceinline__ void ft_prefetch_tile(const FusedArgs& a, uint64_t t, uint32_t tid) {
  if (t >= a.n_ftiles) return;
  const uint32_t T = a.T, R = a.R;
  const uint32_t s2 = a.tile_stage[t];
  const uint32_t p02 = ((uint32_t)t - a.st_tile0[s2]) * T;
  const uint32_t npos2 = a.st_npos[s2];
  const uint32_t np2 = min(T, npos2 - p02);
  const uint64_t rb2 = a.rank_off[s2 * R];
  const uint32_t l4 = (np2 * 4 + 127) / 128 + 1, l2 = (np2 * 2 + 127) / 128 + 1, per_row = 2 * l4 + l2;
  for (uint32_t i = tid; i < R * per_row; i += FT_NT) {
    const uint32_t row = i / per_row, j = i - row * per_row;
    const uint64_t g = rb2 + (uint64_t)row * npos2 + p02;
    const char* col0;
    const char* ptr;
    const char* pe;  // end of the row's segment: a line is fetched only if it holds a byte before it
    uint64_t lim;
    if (j < l4) { col0 = reinterpret_cast<const char*>(a.dur); ptr = reinterpret_cast<const char*>(a.dur + g) + 128ull * j; pe = reinterpret_cast<const char*>(a.dur + g + np2); lim = 4 * a.n_events; }
    else if (j < 2 * l4) { col0 = reinterpret_cast<const char*>(a.comm); ptr = reinterpret_cast<const char*>(a.comm + g) + 128ull * (j - l4); pe = reinterpret_cast<const char*>(a.comm + g + np2); lim = 4 * a.n_events; }
    else { col0 = reinterpret_cast<const char*>(a.kind); ptr = reinterpret_cast<const char*>(a.kind + g) + 128ull * (j - 2 * l4); pe = reinterpret_cast<const char*>(a.kind + g + np2); lim = 2 * a.n_events; }
    if ((uint64_t)(ptr - col0) < lim && (reinterpret_cast<uintptr_t>(ptr) & ~(uintptr_t)127) < reinterpret_cast<uintptr_t>(pe))
      asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
  }
}

template <int P, int NRB>
__global__ void __launch_bounds__(FT_NT, FT_MINB) k_fused_t(FusedArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const uint32_t T = a.T, R = a.R, TP = (uint32_t)a.TP, DP = (uint32_t)a.DP, G = a.G;
  const uint32_t SW = T / 32 + 2, E = TP + DP, NCRM = a.NCRM, RP = R + 1;
  const uint32_t GS = G | 1u, ES = E | 1u;  // odd shared-memory strides (bank-conflict-free columns)
  constexpr uint32_t nrb = NRB;        // row blocks (lane l owns rows l + 32k, k < NRB); R <= 32*NRB
  const uint32_t tpsh = __ffs(TP) - 1;  // TP is a power of two here
  // ---- shared memory carve-up: host-computed byte offsets from smem_raw (fused_t_layout), so every
  // array stays in the shared address space and no per-use offset arithmetic is rematerialised
  uint32_t* sd = reinterpret_cast<uint32_t*>(smem_raw);                              // T x (R+1), position-major
  unsigned long long* rcb = reinterpret_cast<unsigned long long*>(smem_raw + a.o_rcb);
  unsigned long long* coffr = reinterpret_cast<unsigned long long*>(smem_raw + a.o_coffr);
  uint32_t* sinst = reinterpret_cast<uint32_t*>(smem_raw + a.o_sinst);
  uint32_t* sbits = reinterpret_cast<uint32_t*>(smem_raw + a.o_sbits);
  uint32_t* sedge = reinterpret_cast<uint32_t*>(smem_raw + a.o_sedge);
  uint32_t* rcs = reinterpret_cast<uint32_t*>(smem_raw + a.o_rcs);
  uint32_t* rsum = reinterpret_cast<uint32_t*>(smem_raw + a.o_rsum);
  uint32_t* gsum = reinterpret_cast<uint32_t*>(smem_raw + a.o_gsum);
  uint32_t* sjoin = reinterpret_cast<uint32_t*>(smem_raw + a.o_sjoin);
  uint32_t* slate = reinterpret_cast<uint32_t*>(smem_raw + a.o_slate);
  uint32_t* rslow = reinterpret_cast<uint32_t*>(smem_raw + a.o_rslow);
  uint32_t* pa = reinterpret_cast<uint32_t*>(smem_raw + a.o_pa);
  uint32_t* pb = reinterpret_cast<uint32_t*>(smem_raw + a.o_pb);
  uint32_t* vd = reinterpret_cast<uint32_t*>(smem_raw + a.o_vd);
  uint16_t* pk = reinterpret_cast<uint16_t*>(smem_raw + a.o_pk);
  uint16_t* lst = reinterpret_cast<uint16_t*>(smem_raw + a.o_lst);
  uint16_t* cl = reinterpret_cast<uint16_t*>(smem_raw + a.o_cl);
  uint8_t* pcode = reinterpret_cast<uint8_t*>(smem_raw + a.o_pcode);
  // per comm position (indexed by its in-tile comm index): p | class << 14 | deferred << 16 | role << 17,
  // occurrence index k, compute index j of the position, j of the previous comm position; global iteration
  uint4* cinf = reinterpret_cast<uint4*>(smem_raw + a.o_cinf);
  uint32_t* citp = reinterpret_cast<uint32_t*>(smem_raw + a.o_citp);
  __shared__ uint32_t kbase[ROLES];
  __shared__ uint32_t nlist[4];
  __shared__ int32_t dpos;
  __shared__ uint32_t bad, anyslow;

  const uint32_t tile = blockIdx.x;
  const uint32_t tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
  const uint32_t s = a.tile_stage[tile];
  const uint32_t p0 = (tile - a.st_tile0[s]) * T;
  const uint32_t npos = a.st_npos[s];
  const uint32_t np = min(T, npos - p0);
  const uint32_t sbase = s * R;
  const uint64_t n = a.n_ftiles;
  const uint64_t rbase = a.rank_off[sbase];
  const uint32_t j0 = a.ft_base[(uint64_t)ROLES * n + tile];
  const uint32_t m0 = a.ft_base[(uint64_t)(ROLES + 1) * n + tile];
  const uint32_t it0 = a.ft_base[(uint64_t)(ROLES + 2) * n + tile];  // shard-local iteration (citer index)
  const uint32_t itg0 = it0 + a.it_off;  // global iteration: windows, sit, p2p_iter
  const uint32_t jp0 = a.ft_base[(uint64_t)(ROLES + 3) * n + tile];
  const uint32_t wb = j0 >> 5;
  const uint32_t w_tile = win_of(a, itg0);
  const uint32_t ncr = a.ncroles[s];

  // a tile that failed the template verification voids the whole pass (the call reruns the general
  // path): tiles that start after that return at once. One thread reads the flag and the CTA follows
  // its value (another CTA may set it between two threads' reads: every thread must agree)
  {
    __shared__ uint32_t s_void;
    if (tid == 0) s_void = *((volatile const unsigned*)&a.cnt->overflow) & NOT_SPMD;
    __syncthreads();
    if (s_void) return;
  }
  // L2 prefetch of this tile's rows at kernel start: the DRAM requests are in flight while the tables
  // and template info below are set up, so the load pass finds them in L2 (a hint only)
  if (a.pf_own) ft_prefetch_tile(a, tile, tid);
  // ---- (0) tables and template info
  if (tid < ROLES) kbase[tid] = a.ft_base[(uint64_t)tid * n + tile];
  if (tid < 4) nlist[tid] = 0;
  if (tid == 0) { dpos = -1; bad = 0; anyslow = 0; }
  for (uint32_t i = tid; i < R * SW; i += FT_NT) sbits[i] = 0;
  for (uint32_t i = tid; i < R * ES; i += FT_NT) sedge[i] = 0;
  for (uint32_t i = tid; i < 4 * R; i += FT_NT) rsum[i] = 0;
  for (uint32_t i = tid; i < 2 * (DP + TP); i += FT_NT) gsum[i] = 0;
  for (uint32_t i = tid; i < R; i += FT_NT) { sjoin[i] = 0; slate[i] = 0; coffr[i] = a.comm_off[sbase + i]; }
  for (uint32_t i = tid; i < R * ncr; i += FT_NT) {
    const uint32_t row = i / ncr, ro = i - row * ncr;
    const uint32_t cid = a.role_comm[(uint64_t)(sbase + row) * CROLES + ro];
    rcs[row * NCRM + ro] = cid;
    rcb[row * NCRM + ro] = a.ch_base[cid];
  }
  __syncthreads();  // nlist / dpos initialised before the position loop below
  for (uint32_t p = tid; p < T; p += FT_NT) {
    if (p >= np) { pa[p] = 0; pb[p] = 0; pk[p] = 0; vd[p] = 0; pcode[p] = 4; continue; }
    const uint32_t A = a.posA[(uint64_t)tile * T + p], B = a.posB[(uint64_t)tile * T + p];
    const uint16_t K = a.posK[(uint64_t)tile * T + p];
    pa[p] = A; pb[p] = B; pk[p] = K;
    const uint32_t ty = (B >> 25) & 7u, role = (B >> 20) & 31u;
    const bool isc = (K & 7u) == 0;
    const uint32_t li = isc ? 0u : (ty == TY_TP ? 1u : (ty == TY_DP ? 2u : 3u));
    pcode[p] = (uint8_t)li;
    const uint32_t sl = atomicAdd(&nlist[li], 1u);
    lst[li * T + sl] = (uint16_t)p;
    if (isc) {
      vd[p] = 0;
    } else {
      const uint32_t mr = (A >> 10) & 1023u;
      cl[mr] = (uint16_t)(p | ((li - 1u) << 14));
      vd[p] = role < 16 ? (1u | (role << 2)) : (2u | ((uint32_t)(((int)(role & 7u) - 4) * (int)R + 0x100000) << 2));
      const bool def = ((A >> 30) & 1u) && li < 3 && a.mode == 0 && jp0 < j0;
      if (def) dpos = (int32_t)p;
      cinf[mr] = make_uint4(p | ((li - 1u) << 14) | (def ? 1u << 16 : 0u) | (role << 17), kbase[role] + ((B >> 10) & 1023u),
                            j0 + (A & 1023u), ((A >> 30) & 1u) ? jp0 : j0 + ((A >> 20) & 1023u));
      citp[mr] = itg0 + (B & 1023u);
    }
  }
  __syncthreads();
  // L2 prefetch of the payload (and the sender's meta) word of every P2P event of the tile: the phase-B
  // cross units gather them; requested here, the DRAM fetches overlap the load pass below
  if (a.pf_p2p && !a.p2p_defer) {
    const uint32_t nx = nlist[3];
    for (uint32_t i = tid; i < nx * R; i += FT_NT) {
      const uint32_t xi = fdiv(i, a.fR), row = i - xi * R;
      const uint32_t p = lst[3 * T + xi];
      const uint32_t role = (pb[p] >> 20) & 31u;
      if (role < 16) continue;
      const uint64_t e = rbase + (uint64_t)row * npos + p0 + p;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a.pay + e));
      if ((role >> 3) & 1u) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.meta + e));
    }
  }
  // ---- (1) load every rank row of the tile: warps over rows, lanes along positions (fully coalesced),
  // two rows in flight per warp; verify kind_op / comm against the template, transpose into sd[p][row]
  {
    bool mis = false;
    const uint32_t* rcsb = rcs;
    auto check_store = [&](uint32_t row, uint32_t pbase, uint32_t kk0, uint32_t kk1, const uint32_t (&cm)[4],
                           const uint32_t (&du)[4]) {
      const uint2 tk = *reinterpret_cast<const uint2*>(pk + pbase);
      const uint4 v4 = *reinterpret_cast<const uint4*>(vd + pbase);
      const uint32_t dvd[4] = {v4.x, v4.y, v4.z, v4.w};
      mis |= (kk0 != tk.x) | (kk1 != tk.y);
      const uint32_t r = sbase + row;
      const uint32_t* rc = rcsb + row * NCRM;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t t = dvd[i] & 3u, x = dvd[i] >> 2;
        const uint32_t e1 = rc[t == 1 ? x : 0u];
        mis |= (t != 0) & (cm[i] != (t == 1 ? e1 : r + x - 0x100000u));
        if (pbase + i < np) sd[(pbase + i) * RP + row] = du[i];
      }
    };
    auto load4 = [&](uint32_t row, uint32_t pbase, uint32_t& kk0, uint32_t& kk1, uint32_t (&cm)[4], uint32_t (&du)[4]) {
      const uint64_t g = rbase + (uint64_t)row * npos + p0 + pbase;
      if (a.aligned && pbase + 4 <= np) {
        const uint2 kv = __ldg(reinterpret_cast<const uint2*>(a.kind + g));
        const uint4 cv = __ldg(reinterpret_cast<const uint4*>(a.comm + g));
        const uint4 dv4 = __ldg(reinterpret_cast<const uint4*>(a.dur + g));
        kk0 = kv.x; kk1 = kv.y;
        cm[0] = cv.x; cm[1] = cv.y; cm[2] = cv.z; cm[3] = cv.w;
        du[0] = dv4.x; du[1] = dv4.y; du[2] = dv4.z; du[3] = dv4.w;
      } else {
        kk0 = kk1 = 0;
        for (int i = 0; i < 4; ++i) { cm[i] = 0; du[i] = 0; }
        for (uint32_t i = 0; i < 4 && pbase + i < np; ++i) {
          if (i < 2) kk0 |= (uint32_t)a.kind[g + i] << (16 * i); else kk1 |= (uint32_t)a.kind[g + i] << (16 * (i - 2));
          cm[i] = a.comm[g + i];
          du[i] = a.dur[g + i];
        }
      }
    };
    // a warp covers 4*lpr positions of 32/lpr rows (lpr = T/4 lanes per row when T < 128)
    const uint32_t lpr = T >= 128 ? 32u : T / 4u, rpw = 32u / lpr, rstep = FT_NW * rpw;
    const uint32_t rsub = lane / lpr, lpos = lane % lpr;
#if defined(MS_EXP_SKIP) && (MS_EXP_SKIP & 32)
    if (R == 0)  // timing experiment only (results invalid)
#endif
    for (uint32_t pq = 0; pq < np; pq += 4 * lpr) {
      const uint32_t pbase = pq + lpos * 4;
      const bool pin = pbase < np;
      uint32_t row = wid * rpw + rsub;
      for (; row + rstep < R; row += 2 * rstep) {  // two rows per iteration
        uint32_t ka0, ka1, kb0, kb1, cma[4], cmb[4], dua[4], dub[4];
        if (pin) { load4(row, pbase, ka0, ka1, cma, dua); load4(row + rstep, pbase, kb0, kb1, cmb, dub); }
        if (pin) { check_store(row, pbase, ka0, ka1, cma, dua); check_store(row + rstep, pbase, kb0, kb1, cmb, dub); }
      }
      for (; row < R; row += rstep) {
        uint32_t ka0, ka1, cma[4], dua[4];
        if (pin) { load4(row, pbase, ka0, ka1, cma, dua); check_store(row, pbase, ka0, ka1, cma, dua); }
      }
    }
    if (__any_sync(0xFFFFFFFFu, mis) && lane == 0) bad = 1;
  }
  __syncthreads();
  // L2 prefetch of the rows of a tile ahead (blocks start roughly in index order, so tile + pf_dist is
  // loaded soon on some SM): its DRAM traffic overlaps this tile's compute phases instead of stalling
  // that CTA's load pass. A hint only: no result depends on it.
  if (a.pf_dist) ft_prefetch_tile(a, (uint64_t)tile + a.pf_dist, tid);
#if defined(MS_EXP_SKIP) && (MS_EXP_SKIP & 128)
  // timing experiment only (results invalid): a constant tile, so the compute phases cost the same
  // with (bit 128) or without (bits 128 + 32) the row loads
  for (uint32_t i = tid; i < np * RP; i += FT_NT) sd[i] = 1000u;
  __syncthreads();
#endif
  if (bad) { if (tid == 0) atomicOr(&a.cnt->overflow, NOT_SPMD); return; }
  // ---- (2) phase A: stage 1. Exact quick reject per DP group: den*max <= num*min -> nobody slow.
  const uint32_t nc = nlist[0];
#if defined(MS_EXP_SKIP) && (MS_EXP_SKIP & 16)
  if (R == 0)  // timing experiment only (results invalid)
#endif
  if (DP >= 2) {
    bool sl_any = false;
    for (uint32_t i = wid; i < nc; i += FT_NW) {
      const uint32_t p = lst[i];
      const uint32_t* col = sd + p * RP;
      uint32_t mn = 0xFFFFFFFFu, mx = 0;
#pragma unroll
      for (int k = 0; k < NRB; ++k) {
        const uint32_t row = lane + 32u * k;
        if (row < R) { const uint32_t v = col[row]; mn = min(mn, v); mx = max(mx, v); }
      }
      for (uint32_t m = TP; m < 32; m <<= 1) {
        mn = min(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, m));
        mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, m));
      }
      const bool maybe = (unsigned long long)a.slow_den * mx > (unsigned long long)a.slow_num * mn;
      const unsigned need = __ballot_sync(0xFFFFFFFFu, lane < TP && (maybe || a.want_ref));
      if (need) {  // warp-uniform: the rare full LOO path is branched around, not predicated
        if ((need >> lane) & 1u) loo_group<P>(a, col, lane, TP, DP, j0 + (pa[p] & 1023u), sbits, SW, wb, sbase, sl_any);
      }
    }
    if (sl_any) anyslow = 1;
  }
  for (uint32_t p = tid; p < np; p += FT_NT) {
    if (!(pa[p] >> 31)) continue;
    const uint32_t v = j0 + (pa[p] & 1023u) + ((pk[p] & 7u) == 0 ? 1u : 0u);
    const uint32_t itp = it0 + (pb[p] & 1023u);
    for (uint32_t row = 0; row < R; ++row) a.citer[(uint64_t)(sbase + row) * a.NIT1 + itp + 1] = v;
  }
  __syncthreads();
  const bool tslow = anyslow != 0;
  if (tslow)
    for (uint32_t row = tid; row < R; row += FT_NT) {
      uint32_t o = 0;
      for (uint32_t w = 0; w < SW; ++w) o |= sbits[row * SW + w];
      rslow[row] = o != 0;
    }
  __syncthreads();
  // ---- (3) phase B: one warp per comm position
  const uint32_t ncm = nlist[1] + nlist[2] + nlist[3];
  for (uint32_t un = wid; un < ncm * NRB; un += FT_NW) {  // unit = (comm position, row block)
    const uint32_t jj = un / NRB, kb = un - jj * NRB;
    const uint4 cd = cinf[jj];
    const uint32_t p = cd.x & 0x3FFFu, cls = (cd.x >> 14) & 3u;  // 0 TP, 1 DP, 2 cross
    if (cls == 1 && kb != 0) continue;  // a DP group spans every row block: one unit handles it
#if defined(MS_EXP_SKIP) && (MS_EXP_SKIP & 1)
    if (cls == 0) continue;  // timing experiment only (results invalid)
#endif
    const uint32_t role = (cd.x >> 17) & 31u;
    const uint32_t itp = citp[jj];
    uint32_t* col = sd + p * RP;
    if (cls == 2) {
      const uint32_t kk = cd.y;
      {
        const uint32_t row = lane + 32 * kb;
        if (row >= R) continue;
        const uint32_t r = sbase + row;
        uint64_t inst, si;
        uint32_t pay = 0, warm = 0;
        if (role < 16) {
          const uint32_t cid = rcs[row * NCRM + role];
          const uint32_t nm = (uint32_t)(a.coff[cid + 1] - a.coff[cid]);
          inst = rcb[row * NCRM + role] + kk;
          si = a.ch_slot[cid] + (uint64_t)kk * nm + a.role_slot[(uint64_t)r * CROLES + role];
        } else {  // a P2P instance's send / receive slots sit at p2p_slot0 + 2 (inst - p2p_inst0) + 0 / 1
          const bool send = (role >> 3) & 1u;
          const uint64_t e = rbase + (uint64_t)row * npos + p0 + p;
          const uint32_t rb = a.p2p_rbase[(uint64_t)r * 16 + (role - 16)];
          if (rb == NONE32) {  // no such link: the trace is not what the template says
#ifdef MS_DEBUG_CHECKS
            printf("k_fused_t: row %u role %u has no P2P channel (tile %u)\n", row, role, tile);
#endif
            atomicOr(&a.cnt->overflow, NOT_SPMD);
            continue;
          }
          inst = (uint64_t)rb + kk;
          si = a.p2p_slot0 + 2 * (inst - a.p2p_inst0) + (send ? 0 : 1);
#if defined(MS_EXP_SKIP) && (MS_EXP_SKIP & 1024)
          if (R == 0)  // timing experiment only (results invalid)
#endif
          if (a.p2p_defer) {
            pay = p0 + p;  // the event's position in its rank: k_cross_reduce gathers payload and warm-up bit
          } else {
            pay = a.pay[e];
            if (send) warm = ((uint32_t)a.meta[e] >> 14) & 1u;
          }
        }
#if defined(MS_EXP_SKIP) && (MS_EXP_SKIP & 256)
        if (R == 0)  // timing experiment only (results invalid)
#endif
        a.slots[si] = make_uint4(col[row], (uint32_t)(coffr[row] + m0 + jj), slot_z(itp, pk[p], warm), pay);
        col[row] = (uint32_t)inst;  // cross positions: the tile now holds the instance id
      }
      continue;
    }
    const bool istp = cls == 0;
    const uint32_t win = win_of(a, itp);
    const uint32_t clsid = istp ? 1u : 2u;
    const bool elig = (a.classes >> (clsid - 1)) & 1u;
    const bool isdef = (cd.x >> 16) & 1u;
    const bool chk = elig && (a.mode || tslow || isdef);
    const uint32_t jp = cd.z;
    const uint32_t jprev = cd.w;
    const uint32_t kinst = cd.y;
    // one group instance: min / max / last arriver (lowest slot with the min) / tie count, then the
    // members' waits, wait-for edges and stage-2 counters
    auto apply = [&](uint32_t row, uint32_t d, uint32_t mn, uint32_t mx, uint32_t lastrow, uint32_t slot, uint32_t g,
                     uint32_t row0, bool leader, uint32_t nat) {
      const uint32_t last = sbase + lastrow;
      const bool islast = row == lastrow;
      if (leader) {
        const uint64_t inst = rcb[row0 * NCRM + role] + kinst;
#if defined(MS_EXP_SKIP) && (MS_EXP_SKIP & 512)
        if (R == 0)  // timing experiment only (results invalid)
#endif
        a.rec[inst] = make_uint4(mn, mx, last, (SCAN_F_COMPLETE | SCAN_F_KIND_OK | SCAN_F_PAYLOAD_OK | SCAN_F_VALID |
                                                (nat == 1 ? SCAN_F_UNIQUE_LAST : 0u)) | (clsid << 8));
        sinst[p * GS + g] = (uint32_t)inst;
        const uint32_t gi = istp ? g : DP + g;
        add64_lohi(&gsum[gi], &gsum[DP + TP + gi], mn);
      }
      const uint32_t wait = d - mn;
      col[row] = wait;  // in-block comm positions now hold the wait
      if (!islast && (unsigned long long)wait > a.wait_margin) {
        if (win == w_tile) {
          const uint32_t old = atomicAdd(&sedge[row * ES + slot], wait);
          if (old + wait < old)
            atomicAdd(&a.ew[(uint64_t)w_tile * a.nnz_tot + a.eidx[(uint64_t)(sbase + row) * E + slot]], 1ull << 32);
        } else {
          atomicAdd(&a.ew[(uint64_t)win * a.nnz_tot + a.eidx[(uint64_t)(sbase + row) * E + slot]], (unsigned long long)wait);
        }
      }
      if (!chk) return;
      const bool lt = islast && nat == 1 && (unsigned long long)(mx - mn) > a.late_margin;
      if (isdef) {
        if (lt) atomicOr(&a.dlate[(uint64_t)tile * ((R + 31) / 32) + row / 32], 1u << (row & 31));
        return;
      }
      const bool pslow = a.mode != 0 || (rslow[row] && sbits_any(sbits + row * SW, wb, jprev, jp));
      if (!pslow) return;
      if (win == w_tile) { atomicAdd(&sjoin[row], 1u); if (lt) atomicAdd(&slate[row], 1u); }
      else {
        const uint32_t r = sbase + row;
        atomicAdd(&a.wl_joined[(uint64_t)win * a.W + r], 1u);
        if (lt) atomicAdd(&a.wl_late[(uint64_t)win * a.W + r], 1u);
      }
    };
    if (istp) {
      const uint32_t gm = TP >= 32 ? 0xFFFFFFFFu : (((1u << TP) - 1u) << (lane & ~(TP - 1u)));
      {
        const uint32_t k = kb;
        const uint32_t row = lane + 32u * k;
        const bool valid = row < R;
        const uint32_t d = valid ? col[row] : 0xFFFFFFFFu;
        uint32_t mn = d, mx = valid ? d : 0u;
        for (uint32_t m = 1; m < TP; m <<= 1) {
          mn = min(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, m));
          mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, m));
        }
        const unsigned eq = __ballot_sync(0xFFFFFFFFu, valid && d == mn) & gm;
        const uint32_t ls = eq ? (uint32_t)(__ffs(eq) - 1) : 0u;
        if (valid) {
          const uint32_t g = row >> tpsh;
          apply(row, d, mn, mx, ls + 32u * k, ls & (TP - 1u), g, g << tpsh, (lane & (TP - 1u)) == 0, __popc(eq));
        }
      }
    } else {
      uint32_t mn = 0xFFFFFFFFu, mx = 0;
#pragma unroll
      for (uint32_t k = 0; k < nrb; ++k) {
        const uint32_t row = lane + 32u * k;
        if (row < R) { const uint32_t d = col[row]; mn = min(mn, d); mx = max(mx, d); }
      }
      for (uint32_t m = TP; m < 32; m <<= 1) {
        mn = min(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, m));
        mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, m));
      }
      uint32_t lsd = 0xFFFFFFFFu, nat = 0;  // lowest DP index with d == min, tie count
#pragma unroll
      for (uint32_t k = 0; k < nrb; ++k) {
        const uint32_t row = lane + 32u * k;
        if (row < R && col[row] == mn) { lsd = min(lsd, row >> tpsh); ++nat; }
      }
      for (uint32_t m = TP; m < 32; m <<= 1) {
        lsd = min(lsd, __shfl_xor_sync(0xFFFFFFFFu, lsd, m));
        nat += __shfl_xor_sync(0xFFFFFFFFu, nat, m);
      }
#pragma unroll
      for (uint32_t k = 0; k < nrb; ++k) {
        const uint32_t row = lane + 32u * k;
        if (row >= R) break;
        const uint32_t g = row & (TP - 1u);
        apply(row, col[row], mn, mx, g + (lsd << tpsh), TP + lsd, g, g, row < TP, nat);
      }
    }
  }
  __syncthreads();
  // ---- (4) flush: coalesced per-rank inst / wait rows; flat (row, comm position) pairs over all
  // threads (a tile holds a few dozen comm positions: warp-per-row left most lanes idle)
#if defined(MS_EXP_SKIP) && (MS_EXP_SKIP & 2)
  if (R == 0)  // timing experiment only (results invalid)
#endif
  if (ncm) {
    const FDiv fn = fdiv_make(ncm);  // exact for R * ncm < 2^22
    for (uint32_t idx = tid; idx < R * ncm; idx += FT_NT) {
      const uint32_t row = fdiv(idx, fn), j = idx - row * ncm;
      const uint32_t cv = cl[j];
      const uint32_t p = cv & 0x3FFFu, cls = cv >> 14;
      const uint32_t v = sd[p * RP + row];
      const uint32_t gi = cls == 0 ? row >> tpsh : row & (TP - 1u);
      const uint64_t o = coffr[row] + m0 + j;
      if (cls < 2) {
        a.inst_c[o] = sinst[p * GS + gi];
        a.wait_c[o] = v;
      } else {
        a.inst_c[o] = v;  // cross positions: the tile holds the instance id
        a.wait_c[o] = 0;  // placeholder until k_xwait_scatter: no holes, so no partial-sector (read-modify-write) stores
      }
    }
  }
  // per-rank sums from the tile (compute positions hold durations, in-block comm positions hold waits):
  // warp = (row block, position slice), lane = row -> conflict-free column reads, register sums
  {
    constexpr uint32_t NSL = FT_NW / NRB;  // position slices per row block
    const uint32_t rb = wid % NRB, sl = wid / NRB;
    const uint32_t row = rb * 32 + lane;
    const uint32_t plo = sl * ((np + NSL - 1) / NSL), phi = min(np, plo + (np + NSL - 1) / NSL);
    unsigned long long sc = 0, sw = 0;
#if defined(MS_EXP_SKIP) && (MS_EXP_SKIP & 4)
    if (R == 0)  // timing experiment only (results invalid)
#endif
    if (row < R)
      for (uint32_t p = plo; p < phi; ++p) {
        const uint32_t pc = pcode[p];
        const uint32_t v = sd[p * RP + row];
        if (pc == 0) sc += v; else if (pc < 3) sw += v;
      }
    if (row < R) {
      if (sc) add64_lohi(&rsum[4 * row], &rsum[4 * row + 1], sc);
      if (sw) add64_lohi(&rsum[4 * row + 2], &rsum[4 * row + 3], sw);
    }
  }
  __syncthreads();
  // stage-1 counters per (window, rank)
  const uint32_t it_last = itg0 + (np ? (pb[np - 1] & 1023u) : 0u);
  const bool one_window = !a.wi || (win_of(a, itg0) == win_of(a, it_last));
  if (DP >= 2 && nc) {
    if (one_window) {
      for (uint32_t row = tid; row < R; row += FT_NT) {
        const uint32_t r = sbase + row;
        uint32_t sl = 0;
        if (tslow) for (uint32_t w = 0; w < SW; ++w) sl += __popc(sbits[row * SW + w]);
        atomicAdd(&a.wd_total[(uint64_t)w_tile * a.W + r], nc);
        if (sl) atomicAdd(&a.wd_slow[(uint64_t)w_tile * a.W + r], sl);
      }
    } else {
      for (uint32_t i = tid; i < R * nc; i += FT_NT) {
        const uint32_t row = i / nc, p = lst[i - row * nc], r = sbase + row;
        const uint32_t win = win_of(a, itg0 + (pb[p] & 1023u));
        const uint32_t j = j0 + (pa[p] & 1023u);
        atomicAdd(&a.wd_total[(uint64_t)win * a.W + r], 1u);
        if ((sbits[row * SW + (j >> 5) - wb] >> (j & 31)) & 1u) atomicAdd(&a.wd_slow[(uint64_t)win * a.W + r], 1u);
      }
    }
  }
#if defined(MS_EXP_SKIP) && (MS_EXP_SKIP & 64)
  if (R == 0)  // timing experiment only (results invalid)
#endif
  for (uint32_t row = tid; row < R; row += FT_NT) {
    const uint32_t r = sbase + row;
    const uint32_t gt = row >> tpsh, gd = row & (TP - 1u), GO = DP + TP;
    const unsigned long long tr = ((unsigned long long)gsum[GO + gt] << 32 | gsum[gt]) * (TP > 1 ? 1ull : 0ull) +
                                  ((unsigned long long)gsum[GO + DP + gd] << 32 | gsum[DP + gd]) * (DP > 1 ? 1ull : 0ull);
    const unsigned long long comp = (unsigned long long)rsum[4 * row + 1] << 32 | rsum[4 * row];
    const unsigned long long wsum = (unsigned long long)rsum[4 * row + 3] << 32 | rsum[4 * row + 2];
    if (comp) atomicAdd(&a.rk_sum[r], comp);
    if (wsum) atomicAdd(&a.rk_sum[a.W + r], wsum);
    if (tr) atomicAdd(&a.rk_sum[2 * a.W + r], tr);
    if (sjoin[row]) atomicAdd(&a.wl_joined[(uint64_t)w_tile * a.W + r], sjoin[row]);
    if (slate[row]) atomicAdd(&a.wl_late[(uint64_t)w_tile * a.W + r], slate[row]);
  }
#if defined(MS_EXP_SKIP) && (MS_EXP_SKIP & 8)
  if (R == 0)  // timing experiment only (results invalid)
#endif
  {
    // the tile's wait-for edge sums -> global: every edge column index loaded first (independent L2
    // hits in flight together), then the atomics, instead of one dependent load per atomic
    const FDiv fe = fdiv_make(ES);
    constexpr int EK = 8;
    for (uint32_t i0 = tid; i0 < R * ES; i0 += EK * FT_NT) {
      uint32_t v[EK], col[EK];
#pragma unroll
      for (int q = 0; q < EK; ++q) {
        const uint32_t i = i0 + (uint32_t)q * FT_NT;
        v[q] = 0; col[q] = 0;
        if (i < R * ES) {
          const uint32_t row = fdiv(i, fe), slot = i - row * ES;
          if (slot < E) { v[q] = sedge[i]; if (v[q]) col[q] = a.eidx[(uint64_t)(sbase + row) * E + slot]; }
        }
      }
#pragma unroll
      for (int q = 0; q < EK; ++q)
        if (v[q]) atomicAdd(&a.ew[(uint64_t)w_tile * a.nnz_tot + col[q]], (unsigned long long)v[q]);
    }
  }
  if (nc && tslow) {
    const uint32_t w_first = j0 >> 5, w_last = (j0 + nc - 1) >> 5;
    const uint32_t nw = w_last - w_first + 1;
    for (uint32_t i = tid; i < R * nw; i += FT_NT) {
      const uint32_t row = i / nw, w = w_first + (i - row * nw);
      const uint32_t v = sbits[row * SW + (w - wb)];
      if (v) atomicOr(&a.bits[a.bits_off[sbase + row] + w], v);
    }
  }
  if (tid == 0) {
    uint32_t* di = a.dinfo + (uint64_t)tile * 4;
    if (dpos >= 0) {
      const uint32_t p = (uint32_t)dpos;
      const uint32_t ty = (pb[p] >> 25) & 7u;
      di[0] = j0 + (pa[p] & 1023u); di[1] = jp0; di[2] = win_of(a, itg0 + (pb[p] & 1023u)); di[3] = 1u | (ty << 8);
    } else {
      di[3] = 0;
    }
  }
}

static size_t fused_t_layout(uint32_t T, uint32_t R, uint32_t TP, uint32_t DP, uint32_t NCRM, FusedArgs* a) {
  const uint32_t SW = T / 32 + 2, G = TP > DP ? TP : DP, E = TP + DP, RP = R + 1;
  size_t off = 0;
  auto take = [&](size_t bytes, size_t align) { off = (off + align - 1) & ~(align - 1); const size_t o = off; off += bytes; return (uint32_t)o; };
  take((size_t)T * RP * 4, 16);
  const uint32_t o_rcb = take((size_t)R * NCRM * 8, 16), o_coffr = take((size_t)R * 8, 8), o_sinst = take((size_t)T * (G | 1u) * 4, 4);
  const uint32_t o_sbits = take((size_t)R * SW * 4, 4), o_sedge = take((size_t)R * (E | 1u) * 4, 4), o_rcs = take((size_t)R * NCRM * 4, 4);
  const uint32_t o_rsum = take((size_t)R * 16, 4), o_gsum = take((size_t)(DP + TP) * 8, 4), o_sjoin = take((size_t)R * 4, 4);
  const uint32_t o_slate = take((size_t)R * 4, 4), o_rslow = take((size_t)R * 4, 4), o_pa = take((size_t)T * 4, 16);
  const uint32_t o_pb = take((size_t)T * 4, 16), o_vd = take((size_t)T * 4, 16), o_pk = take((size_t)T * 2, 16);
  const uint32_t o_lst = take((size_t)T * 8, 4), o_cl = take((size_t)T * 2, 4), o_pcode = take((size_t)T, 4);
  const uint32_t o_cinf = take((size_t)T * 16, 16), o_citp = take((size_t)T * 4, 4);
  if (a) {
    a->o_rcb = o_rcb; a->o_coffr = o_coffr; a->o_sinst = o_sinst; a->o_sbits = o_sbits; a->o_sedge = o_sedge; a->o_rcs = o_rcs;
    a->o_rsum = o_rsum; a->o_gsum = o_gsum; a->o_sjoin = o_sjoin; a->o_slate = o_slate; a->o_rslow = o_rslow; a->o_pa = o_pa;
    a->o_pb = o_pb; a->o_vd = o_vd; a->o_pk = o_pk; a->o_lst = o_lst; a->o_cl = o_cl; a->o_pcode = o_pcode;
    a->o_cinf = o_cinf; a->o_citp = o_citp;
  }
  return (off + 15) & ~size_t(15);
}

// shared-memory budget per CTA so that FT_MINB CTAs of the transposed kernel fit on one SM
size_t fused_t_smem_cap() { return (size_t)220 * 1024 / FT_MINB; }

// events per tile of the transposed kernel: 32 per thread (16384 at 512 threads; 32768 at the default
// 1024: R = 128 rows x 256 positions on C3, half the per-tile set-up per event of 128 positions)
uint32_t fused_t_tile_events() { return 32u * (uint32_t)FT_NT; }

size_t fused_t_smem_bytes(uint32_t T, uint32_t R, uint32_t TP, uint32_t DP, uint32_t NCRM) {
  return fused_t_layout(T, R, TP, DP, NCRM, nullptr);
}

size_t fused_smem_bytes(uint32_t T, uint32_t R, uint32_t TP, uint32_t DP, uint32_t NCRM) {
  const uint32_t SW = T / 32 + 2, G = TP > DP ? TP : DP;
  size_t b = (size_t)R * T * 4 + (size_t)T * 4 + (size_t)R * 8 + (size_t)R * NCRM * 8 + (size_t)R * 16 +
             (size_t)(DP + TP) * 8 + (size_t)R * (TP + DP) * 8 + (size_t)R * 4 + (size_t)T * G * 4 +
             (size_t)R * SW * 4 + (size_t)R * NCRM * 4 + (size_t)T * 4 * 5 + (size_t)R * 12 + (size_t)T / 4 + 8 +
             (size_t)T * 2 + (size_t)T * 8 + (size_t)T * 2 + 16;
  return (b + 15) & ~size_t(15);
}

// Instance base of the P2P channel behind every (rank, P2P role) -- role 16 + 8 send + stage delta + 4 --
// or NONE32 where the role names no channel, so the fused kernels place a P2P member without the
// per-event bitmap search and channel lookups
__global__ void k_p2p_roles(int W, uint32_t R, uint32_t n_comms, const uint32_t* bitmap, const uint32_t* bitpre,
                            const uint64_t* ch_base, uint32_t* out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (uint32_t)W * 16u) return;
  const uint32_t r = i >> 4, x = i & 15u;
  const bool send = x >> 3;
  const int peer = (int)r + ((int)(x & 7u) - 4) * (int)R;
  uint32_t v = NONE32;
  if (peer >= 0 && peer < W) {
    const uint32_t src = send ? r : (uint32_t)peer, dst = send ? (uint32_t)peer : r;
    const uint32_t xk = src * (uint32_t)W + dst;
    const uint32_t bm = bitmap[xk >> 5];
    if ((bm >> (xk & 31)) & 1u) v = (uint32_t)ch_base[n_comms + bitpre[xk >> 5] + __popc(bm & ((1u << (xk & 31)) - 1u))];
  }
  out[i] = v;
}

int launch_p2p_roles(Ctx& c) {  // c.p2p_rbase sized by alloc_match_buffers
  if (c.n_p2p == 0) return 0;
  const uint32_t n = (uint32_t)c.W * 16u;
  k_p2p_roles<<<(n + 255) / 256, 256, 0, c.stream>>>(c.W, c.FR, c.n_comms, c.bitmap.as<uint32_t>(), c.bitpre.as<uint32_t>(),
                                                     c.ch_base.as<uint64_t>(), c.p2p_rbase.as<uint32_t>());
  return 1;
}

// MS_P2P_DEFER=1: the transposed fused kernel leaves P2P payload / meta to k_cross_reduce (experiment)
bool p2p_defer_on(Ctx& c) {
  static int v = -1;
  if (v < 0) { const char* e = std::getenv("MS_P2P_DEFER"); v = e ? std::atoi(e) : 0; }
  return v == 1 && c.fused_t && !stage_active(c);
}

int launch_fused(Ctx& c) {
  if (stage_active(c)) {  // the persistent TMA-fed kernel (k_stage.cu)
    const int n = launch_stage(c);
    if (n >= 0) return n;
    c.use_stage = false;  // no tensor maps (driver entry point): the transposed kernel, same tile size
  }
  FusedArgs a;
  a.dur = c.d_dur; a.kind = c.d_kind; a.meta = c.d_meta; a.comm = c.d_comm; a.pay = c.d_pay;
  a.rank_off = c.rank_off.as<uint64_t>(); a.TP = c.TP; a.DP = c.DP; a.PP = c.PP; a.W = c.W; a.n_comms = c.n_comms;
  a.T = c.FT; a.R = c.FR; a.n_ftiles = c.n_ftiles; a.G = (uint32_t)std::max(c.TP, c.DP); a.aligned = c.rows_aligned;
  a.aligned8 = c.rows_aligned8;
  a.st_tile0 = c.st_tile0.as<uint32_t>(); a.st_npos = c.st_npos.as<uint32_t>(); a.ft_base = c.ft_base.as<uint32_t>();
  a.tile_stage = c.tile_stage.as<uint8_t>();
  a.fTP = fdiv_make(c.TP); a.fDP = fdiv_make(c.DP); a.fR = fdiv_make(c.FR); a.fG = fdiv_make(c.FT / 4);
  a.fCH = fdiv_make((c.FT + 127) / 128);
  a.posA = c.ft_posA.as<uint32_t>(); a.posB = c.ft_posB.as<uint32_t>(); a.posK = c.ft_posK.as<uint16_t>();
  a.role_comm = c.role_comm.as<uint32_t>(); a.role_slot = c.role_slot.as<uint32_t>();
  a.ncroles = c.ncroles.as<uint32_t>(); a.NCRM = c.NCRM; a.eidx = c.eidx.as<uint32_t>(); a.coff = c.coff.as<uint64_t>();
  a.ch_base = c.ch_base.as<uint64_t>(); a.ch_slot = c.ch_slot.as<uint64_t>(); a.bitmap = c.bitmap.as<uint32_t>();
  a.bitpre = c.bitpre.as<uint32_t>(); a.comm_off = c.r_comm_off.as<uint64_t>(); a.comp_off = c.r_comp_off.as<uint64_t>();
  a.bits_off = c.r_bits_off.as<uint64_t>(); a.inst_c = c.inst_c.as<uint32_t>(); a.wait_c = c.wait_c.as<uint32_t>();
  a.bits = c.bits.as<uint32_t>(); a.cref = c.cref.as<uint32_t>(); a.rec = c.inst_rec.as<uint4>();
  a.slots = c.slots.as<uint4>(); a.p2p_rbase = c.p2p_rbase.as<uint32_t>();
  a.p2p_slot0 = c.p2p_slot0; a.p2p_inst0 = c.p2p_inst0; a.citer = c.citer.as<uint32_t>(); a.NIT1 = c.NIT + 1;
  {  // L2 prefetches of the transposed kernel. Round 1 (512 x 128 tiles, 2 CTAs per SM; k_fused_t ms): none
     // 8.51; own tile at kernel start 8.22; tile pf ahead after the load pass: 96 8.32, 148 8.35, 296 8.93.
     // With 1024 x 256 tiles (one CTA per SM, round 2) every prefetch costs: own tile + P2P words 6.86,
     // own only 6.78, P2P only 6.70, none 6.61 (default); pf 74 / 148 ahead 7.40 / 7.45.
     // MS_FT_PF (distance, 0 = off) / MS_FT_PF_OWN / MS_FT_PF_P2P (0/1) override
    static int pf = -1;
    if (pf < 0) {
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
      const char* e = std::getenv("MS_FT_PF");
      pf = e ? std::atoi(e) : 0;
      (void)sms;
    }
    static int own = -1;
    if (own < 0) { const char* e = std::getenv("MS_FT_PF_OWN"); own = e ? std::atoi(e) : 0; }
    static int pp = -1;
    if (pp < 0) { const char* e = std::getenv("MS_FT_PF_P2P"); pp = e ? std::atoi(e) : 0; }
    a.pf_p2p = (uint32_t)pp;
    a.p2p_defer = p2p_defer_on(c) ? 1u : 0u;
    a.pf_dist = (uint32_t)pf;
    a.pf_own = (uint32_t)own;
    a.n_events = c.N;
  }
  a.nbc_off = c.nbc_off.as<uint64_t>(); a.nbc = c.nbc.as<uint32_t>(); a.nbp = c.nbp.as<uint32_t>();
  a.nbp_n = c.nbp_n.as<uint32_t>(); a.nnz_tot = c.nnz_c + (uint64_t)c.W * PCAP; a.nnz_c = c.nnz_c;
  a.ew = c.ewc.as<unsigned long long>(); a.rk_sum = c.rk_sum.as<unsigned long long>();
  a.wl_joined = c.wl_joined.as<uint32_t>(); a.wl_late = c.wl_late.as<uint32_t>();
  a.wd_total = c.wd_total.as<uint32_t>(); a.wd_slow = c.wd_slow.as<uint32_t>();
  a.dlate = c.dlate.as<uint32_t>(); a.dinfo = c.dinfo.as<uint32_t>();
  a.slow_num = c.dcfg.slow_num; a.slow_den = c.dcfg.slow_den; a.slow_margin = c.dcfg.slow_margin_ns;
  a.wi = c.dcfg.window_iters; a.classes = c.lcfg.stage2_classes; a.mode = c.lcfg.stage2_mode;
  a.it_off = c.it_off;
  a.wi_m = c.dcfg.window_iters > 1 ? (~0ull / c.dcfg.window_iters) + 1ull : 0ull;
  a.late_margin = c.lcfg.late_margin_ns; a.wait_margin = c.lcfg.wait_margin_ns; a.want_ref = c.dcfg.want_ref ? 1 : 0;
  a.cnt = c.counters.as<Counters>();
  if (c.fused_t) {
    const size_t sm = fused_t_layout(c.FT, c.FR, c.TP, c.DP, c.NCRM, &a);
    auto go = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      kern<<<c.n_ftiles, FT_NT, sm, c.stream>>>(a);
    };
    const uint32_t nrb = (c.FR + 31) / 32;
    auto go_p = [&](auto tagP) {
      constexpr int PP_ = decltype(tagP)::value;
      if (nrb <= 1) go(k_fused_t<PP_, 1>);
      else if (nrb <= 2) go(k_fused_t<PP_, 2>);
      else if (nrb <= 4) go(k_fused_t<PP_, 4>);
      else go(k_fused_t<PP_, 8>);
    };
    if (c.DP < 2) go_p(std::integral_constant<int, 1>{});
    else if (c.DP <= 2) go_p(std::integral_constant<int, 2>{});
    else if (c.DP <= 4) go_p(std::integral_constant<int, 4>{});
    else if (c.DP <= 8) go_p(std::integral_constant<int, 8>{});
    else if (c.DP <= 16) go_p(std::integral_constant<int, 16>{});
    else go_p(std::integral_constant<int, 32>{});
    return 1;
  }
  const size_t sm = fused_smem_bytes(c.FT, c.FR, c.TP, c.DP, c.NCRM);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    kern<<<c.n_ftiles, F_NT, sm, c.stream>>>(a);
  };
  if (c.DP < 2) go(k_fused<1>);
  else if (c.DP <= 2) go(k_fused<2>);
  else if (c.DP <= 4) go(k_fused<4>);
  else if (c.DP <= 8) go(k_fused<8>);
  else if (c.DP <= 16) go(k_fused<16>);
  else go(k_fused<32>);
  return 1;
}

// ----------------------------------------------------------------------------- cross-stage instances
// Instances whose members span stage blocks (model-parallel, embedding, P2P, any non TP/DP
// communicator): integrity + decomposition (as k_inst_reduce), then the members' waits,
// per-rank sums and wait-for edges from the slot arrays written by k_fused.
struct XArgs {
  uint64_t n_xinst, NCH; uint32_t n_comms; int W; const uint64_t* xbase;
  const uint64_t* ch_base; const uint64_t* ch_slot; const uint32_t* ch_nmin; const uint64_t* coff; const uint32_t* cmem;
  const uint8_t* ccls; const uint32_t* nsend; const uint32_t* nrecv; const uint32_t* psrc; const uint32_t* pdst;
  const uint32_t* r_nkeys; const uint32_t* r_keys; const uint32_t* r_cnt;
  uint4* slots;  // SlotRec; after the reduction a member slot's x holds that member's wait (instance order)
  uint4* rec; uint32_t* wait_c;
  unsigned long long* lk_key; uint64_t p2p_inst0;  // stage-3 sample key per P2P instance
  const uint64_t* nbc_off; const uint32_t* nbc; const uint32_t* nbp; const uint32_t* nbp_n; uint64_t nnz_tot, nnz_c;
  unsigned long long* ew; unsigned long long* rk_sum; uint32_t wi; unsigned long long wait_margin;
  Counters* cnt;
  const uint32_t* p2p_eslot;  // [n_p2p][2] edge column of src -> dst and dst -> src
  int xb_smem;                // xbase staged in shared memory (NCH + 1 entries)
  const uint64_t* xe_off;     // [n_comms] offset of a cross collective's member x member edge-column table, ~0 = none
  const uint32_t* xe_col;     // table[q * nm + t]: edge column of member q waiting on member t
  // k_stage leaves each P2P member's position within its rank in the slot's w: gather the payload and
  // the sender's warm-up bit here (latency-tolerant grid) instead of between the fused kernel's barriers
  int p2p_pos; const uint32_t* pay; const uint16_t* meta; const uint64_t* rank_off;
};



constexpr uint32_t XBIG = 32;  // cross collectives with more members go to k_cross_big

// warp sum of values < 2^32 (one per lane) as 16-bit halves with single-instruction full-warp
// reductions: each half sums to < 2^21, no overflow
__device__ __forceinline__ unsigned long long warp_sum_small(unsigned long long v) {
  const uint32_t x = (uint32_t)v;
  const uint32_t lo = __reduce_add_sync(0xFFFFFFFFu, x & 0xFFFFu), hi = __reduce_add_sync(0xFFFFFFFFu, x >> 16);
  return (unsigned long long)lo + ((unsigned long long)hi << 16);
}

// edge column of every P2P link direction (the search x_edge would do), once per analysis
__global__ void k_p2p_eslot(uint32_t n_p2p, const uint32_t* psrc, const uint32_t* pdst, const uint64_t* nbc_off,
                            const uint32_t* nbc, const uint32_t* nbp, const uint32_t* nbp_n, uint64_t nnz_c, uint32_t* out) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_p2p) return;
  for (int q = 0; q < 2; ++q) {
    const uint32_t r = q ? pdst[p] : psrc[p], L = q ? psrc[p] : pdst[p];
    const uint64_t nb0 = nbc_off[r], nb1 = nbc_off[r + 1];
    const uint32_t pc = lower_bound_u32(nbc + nb0, (uint32_t)(nb1 - nb0), L);
    out[2 * p + q] = (uint32_t)((pc < nb1 - nb0 && nbc[nb0 + pc] == L)
                                    ? nb0 + pc
                                    : nnz_c + (uint64_t)r * PCAP + lower_bound_u32(nbp + (uint64_t)r * PCAP, nbp_n[r], L));
  }
}

__device__ __forceinline__ void x_edge(const XArgs& a, uint32_t r, uint32_t L, uint32_t win, unsigned long long wait) {
  const uint64_t nb0 = a.nbc_off[r], nb1 = a.nbc_off[r + 1];
  uint64_t idx;
  const uint32_t pc = lower_bound_u32(a.nbc + nb0, (uint32_t)(nb1 - nb0), L);
  if (pc < nb1 - nb0 && a.nbc[nb0 + pc] == L) idx = nb0 + pc;
  else idx = a.nnz_c + (uint64_t)r * PCAP + lower_bound_u32(a.nbp + (uint64_t)r * PCAP, a.nbp_n[r], L);
  atomicAdd(&a.ew[(uint64_t)win * a.nnz_tot + idx], wait);
}

#ifndef MS_XR_MINB
#define MS_XR_MINB 4  // 3 or 2 CTAs per SM (more registers, no spills) measured slower: 0.36 -> 0.40 / 0.51 ms
#endif
__global__ void __launch_bounds__(256, MS_XR_MINB) k_cross_reduce(XArgs a) {
  if (*((volatile unsigned*)&a.cnt->overflow) & NOT_SPMD) return;  // fused results void: general path reruns
  extern __shared__ unsigned long long xb_s[];
  if (a.xb_smem) {
    for (uint64_t q = threadIdx.x; q <= a.NCH; q += blockDim.x) xb_s[q] = a.xbase[q];
    __syncthreads();
  }
  const uint64_t* XB = a.xb_smem ? reinterpret_cast<const uint64_t*>(xb_s) : a.xbase;
  uint32_t inc = 0, kmis = 0, pmis = 0;
  const uint32_t lane = lane_id();
  // each warp walks a contiguous chunk of instances (32 per step): consecutive steps stay in one channel,
  // so the channel search runs only when a step leaves the cached channel
  const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t gw = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint64_t per = ((a.n_xinst + nwarps - 1) / nwarps + 31) & ~31ull;
  const uint64_t wend = min(a.n_xinst, (gw + 1) * per);
  // the warp's current channel, its instance range [beg0, end0) in cross order, and (P2P) its tables
  uint64_t ch0 = 0, beg0 = 1, end0 = 0, ib0 = 0, sl0 = 0, ro_src0 = 0, ro_dst0 = 0;
  uint32_t src0 = 0, dst0 = 0, nsd0 = 0, nrc0 = 0;
  // P2P fast path (whole warp on one link, one window): per-lane sums over the warp's steps on the
  // cached link -- member waits, transfer, wait-for edges src -> dst / dst -> src -- flushed with one
  // atomic each when the warp leaves the link
  unsigned long long acc_w0 = 0, acc_w1 = 0, acc_t = 0, acc_e0 = 0, acc_e1 = 0;
  auto flush_link = [&]() {
    const unsigned long long w0 = warp_sum_u64(acc_w0), w1 = warp_sum_u64(acc_w1), t = warp_sum_u64(acc_t);
    const unsigned long long e0 = warp_sum_u64(acc_e0), e1 = warp_sum_u64(acc_e1);
    if (lane == 0 && ch0 >= a.n_comms) {
      const uint64_t p = ch0 - a.n_comms;
      if (w0) atomicAdd(&a.rk_sum[a.W + src0], w0);
      if (w1) atomicAdd(&a.rk_sum[a.W + dst0], w1);
      if (t) { atomicAdd(&a.rk_sum[2 * a.W + src0], t); atomicAdd(&a.rk_sum[2 * a.W + dst0], t); }
      if (e0) atomicAdd(&a.ew[a.p2p_eslot[2 * p]], e0);
      if (e1) atomicAdd(&a.ew[a.p2p_eslot[2 * p + 1]], e1);
    }
    acc_w0 = acc_w1 = acc_t = acc_e0 = acc_e1 = 0;
  };
  for (uint64_t wbase = gw * per; wbase < wend; wbase += 32) {
    const uint64_t xi = wbase + lane;
    bool act = xi < wend;
    // channel of the warp's first instance; lanes past its end search alone
    if (!(wbase >= beg0 && wbase < end0)) {
      flush_link();
      if (lane == 0) {
        ch0 = upper_bound_u64(XB, a.NCH + 1, wbase) - 1; beg0 = XB[ch0]; end0 = XB[ch0 + 1];
        ib0 = a.ch_base[ch0]; sl0 = a.ch_slot[ch0];
        if (ch0 >= a.n_comms) {
          const uint64_t p = ch0 - a.n_comms;
          src0 = a.psrc[p]; dst0 = a.pdst[p]; nsd0 = a.nsend[p]; nrc0 = a.nrecv[p];
          if (a.p2p_pos) { ro_src0 = a.rank_off[src0]; ro_dst0 = a.rank_off[dst0]; }
        }
      }
      ch0 = __shfl_sync(0xFFFFFFFFu, ch0, 0); beg0 = __shfl_sync(0xFFFFFFFFu, beg0, 0); end0 = __shfl_sync(0xFFFFFFFFu, end0, 0);
      ib0 = __shfl_sync(0xFFFFFFFFu, ib0, 0); sl0 = __shfl_sync(0xFFFFFFFFu, sl0, 0);
      src0 = __shfl_sync(0xFFFFFFFFu, src0, 0); dst0 = __shfl_sync(0xFFFFFFFFu, dst0, 0);
      ro_src0 = __shfl_sync(0xFFFFFFFFu, ro_src0, 0); ro_dst0 = __shfl_sync(0xFFFFFFFFu, ro_dst0, 0);
      nsd0 = __shfl_sync(0xFFFFFFFFu, nsd0, 0); nrc0 = __shfl_sync(0xFFFFFFFFu, nrc0, 0);
    }
    if (ch0 >= a.n_comms) {  // P2P channel: L2 prefetch of the slot sector two steps ahead (same channel)
      const uint64_t xp = xi + 64;
      if (xp < end0 && xp < wend) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.slots + sl0 + 2 * (xp - beg0)));
    }
    uint64_t ch = 0, k = 0, i = 0, slb = 0;
    uint32_t psrc_ = 0, pdst_ = 0, nsd = 0, nrc = 0;
    if (act) {
      if (xi < end0) {
        ch = ch0; k = xi - beg0; i = ib0 + k; slb = sl0; psrc_ = src0; pdst_ = dst0; nsd = nsd0; nrc = nrc0;
      } else {
        ch = upper_bound_u64(XB, a.NCH + 1, xi) - 1;
        k = xi - XB[ch];
        i = a.ch_base[ch] + k; slb = a.ch_slot[ch];
        if (ch >= a.n_comms) {
          const uint64_t p = ch - a.n_comms;
          psrc_ = a.psrc[p]; pdst_ = a.pdst[p]; nsd = a.nsend[p]; nrc = a.nrecv[p];
        }
      }
      if (ch < a.n_comms && a.coff[ch + 1] - a.coff[ch] > XBIG) act = false;  // k_cross_big (lanes over members)
    }
    // one channel across the whole warp (the common case): its members are the same for every lane
    const bool uni = __all_sync(0xFFFFFFFFu, act && ch == ch0);
    const bool isp = ch >= a.n_comms;
    const uint32_t nm = isp ? 2u : (uint32_t)(a.coff[ch + 1] - a.coff[ch]);
    const uint64_t sb = slb + k * nm;
    auto member = [&](uint32_t q) -> uint32_t { return isp ? (q == 0 ? psrc_ : pdst_) : a.cmem[a.coff[ch] + q]; };
    if (uni && isp && !a.wi) {
      // P2P fast path: both slots in one 32-byte sector; complete = both present (ch_nmin = min(sends, recvs))
      const bool h0 = nsd > k, h1 = nrc > k;
      uint4 s0 = make_uint4(0, 0, 0, 0), s1 = s0;
      if (h0) s0 = a.slots[sb];
      if (h1) s1 = a.slots[sb + 1];
      if (a.p2p_pos) {  // the fused pass left each member's position in its rank: gather payload and warm-up bit
        if (h0) {
          const uint64_t e0 = ro_src0 + s0.w;
          s0.w = a.pay[e0];
          s0.z = (s0.z & 0x7FFFFFFFu) | (((uint32_t)a.meta[e0] >> 14) & 1u) << 31;
          reinterpret_cast<uint32_t*>(a.slots + sb)[3] = s0.w;
        }
        if (h1) {
          s1.w = a.pay[ro_dst0 + s1.w];
          reinterpret_cast<uint32_t*>(a.slots + sb + 1)[3] = s1.w;
        }
      }
      uint32_t flags = (s0.z >> 31) ? SCAN_F_WARMUP : 0u, dmin = 0, dmax = 0, last = NONE32;
      if (h0 && h1) {
        flags |= SCAN_F_COMPLETE | SCAN_F_KIND_OK;
        if (s0.w == s1.w) {
          flags |= SCAN_F_PAYLOAD_OK | SCAN_F_VALID;
          dmin = min(s0.x, s1.x); dmax = max(s0.x, s1.x);
          if (s0.x != s1.x) flags |= SCAN_F_UNIQUE_LAST;
          const bool l1 = s1.x < s0.x;  // last arriver: lowest member with the minimum
          last = l1 ? pdst_ : psrc_;
          const uint32_t w0 = s0.x - dmin, w1 = s1.x - dmin;
          acc_w0 += w0; acc_w1 += w1; acc_t += dmin;
          if (l1 && (unsigned long long)w0 > a.wait_margin) acc_e0 += w0;   // src waits on dst
          if (!l1 && (unsigned long long)w1 > a.wait_margin) acc_e1 += w1;  // dst waits on src
        } else {
          ++pmis;
        }
      } else {
        ++inc;
      }
      a.rec[i] = make_uint4(dmin, dmax, last, flags);
      a.lk_key[i - a.p2p_inst0] = lk_sample_key(flags, dmin, s0.w);
      continue;
    }
    auto present = [&](uint32_t q) -> bool {
      if (isp) return (q == 0 ? nsd : nrc) > k;
      const uint32_t m = a.cmem[a.coff[ch] + q];
      const uint32_t C = a.r_nkeys[m];
      const uint32_t p = lower_bound_u32(a.r_keys + (uint64_t)m * RCAP, C, (uint32_t)ch);
      return p < C && a.r_keys[(uint64_t)m * RCAP + p] == (uint32_t)ch && a.r_cnt[(uint64_t)m * RCAP + p] > k;
    };
    uint32_t flags = 0, dmin = 0, dmax = 0, last = NONE32, lsi = 0;
    bool valid = false;
    // a P2P instance's send and receive slots: one 32-byte sector, read once
    uint4 s0 = make_uint4(0, 0, 0, 0), s1 = s0;
    if (act && isp) {
      const bool h0 = nsd > k, h1 = nrc > k;
      if (h0) s0 = a.slots[sb];
      if (h1) s1 = a.slots[sb + 1];
      if (a.p2p_pos) {
        if (h0) {
          const uint64_t e = a.rank_off[member(0)] + s0.w;
          s0.w = a.pay[e];
          s0.z = (s0.z & 0x7FFFFFFFu) | (((uint32_t)a.meta[e] >> 14) & 1u) << 31;
          reinterpret_cast<uint32_t*>(a.slots + sb)[3] = s0.w;
        }
        if (h1) {
          s1.w = a.pay[a.rank_off[member(1)] + s1.w];
          reinterpret_cast<uint32_t*>(a.slots + sb + 1)[3] = s1.w;
        }
      }
      if (s0.z >> 31) flags |= SCAN_F_WARMUP;  // the sender's flag (0 when the send is absent)
    }
    auto sdur = [&](uint32_t q) -> uint32_t { return isp ? (q ? s1.x : s0.x) : a.slots[sb + q].x; };
    auto sit = [&](uint32_t q) -> uint32_t { return (isp ? (q ? s1.z : s0.z) : a.slots[sb + q].z) & SLOT_IT_MASK; };
    if (act) {
      if (k < a.ch_nmin[ch]) {
        flags |= SCAN_F_COMPLETE;
        bool kind_ok = true, pay_ok = true;
        if (!isp) {
          const uint32_t k0 = slot_kind(a.slots[sb].z);
          for (uint32_t q = 1; q < nm; ++q) if (slot_kind(a.slots[sb + q].z) != k0) kind_ok = false;
        } else {
          pay_ok = s0.w == s1.w;
        }
        if (kind_ok) flags |= SCAN_F_KIND_OK; else ++kmis;
        if (pay_ok) flags |= SCAN_F_PAYLOAD_OK; else ++pmis;
        if (kind_ok && pay_ok) {
          valid = true;
          flags |= SCAN_F_VALID;
          dmin = NONE32;
          uint32_t ls = 0, nat = 0;
          for (uint32_t q = 0; q < nm; ++q) {
            const uint32_t d = sdur(q);
            if (d < dmin) { dmin = d; ls = q; nat = 1; } else if (d == dmin) ++nat;
            dmax = max(dmax, d);
          }
          if (nat == 1) flags |= SCAN_F_UNIQUE_LAST;
          last = member(ls);
          lsi = ls;
        }
      } else {
        ++inc;
      }
      a.rec[i] = make_uint4(dmin, dmax, last, flags | ((isp ? 0u : a.ccls[ch]) << 8));
      if (isp) a.lk_key[i - a.p2p_inst0] = lk_sample_key(flags, dmin, s0.w);
    }
    if (uni) {
      // aggregated per-member sums (members identical across lanes); the wait-for edge too when
      // every contributing lane has the same target and window (always for a P2P link: the
      // target is the other endpoint), else one atomic per lane
      for (uint32_t q = 0; q < nm; ++q) {
        unsigned long long w = 0, t = 0;
        bool eg = false;
        uint32_t ewin = 0, ewait = 0;
        if (act && valid) {  // (a member's wait, duration - dmin, is recomputed where it is exported: k_xwait_scatter)
          const uint32_t m = member(q);
          const uint32_t wait = sdur(q) - dmin;
          w = wait; t = dmin;
          if (m != last && (unsigned long long)wait > a.wait_margin) {
            eg = true; ewait = wait; ewin = a.wi ? sit(q) / a.wi : 0;
          }
        }
        const unsigned em = __ballot_sync(0xFFFFFFFFu, eg);
        if (em) {
          const int L0 = __ffs(em) - 1;
          const uint32_t tl = __shfl_sync(0xFFFFFFFFu, last, L0), tw = __shfl_sync(0xFFFFFFFFu, ewin, L0);
          const uint32_t tli = __shfl_sync(0xFFFFFFFFu, lsi, L0);
          if (__all_sync(0xFFFFFFFFu, !eg || (last == tl && ewin == tw))) {
            const unsigned long long ws = warp_sum_small(eg ? (unsigned long long)ewait : 0ull);
            if (lane == (uint32_t)L0) {
              if (isp) atomicAdd(&a.ew[(uint64_t)tw * a.nnz_tot + a.p2p_eslot[2 * (ch - a.n_comms) + q]], ws);
              else if (a.xe_off[ch] != ~0ull) atomicAdd(&a.ew[(uint64_t)tw * a.nnz_tot + a.xe_col[a.xe_off[ch] + (uint64_t)q * nm + tli]], ws);
              else x_edge(a, member(q), tl, tw, ws);
            }
          } else if (eg) {
            x_edge(a, member(q), last, ewin, ewait);
          }
        }
        w = warp_sum_small(w); t = warp_sum_small(t);
        if (lane == 0) {
          const uint32_t m = member(q);
          if (w) atomicAdd(&a.rk_sum[a.W + m], w);
          if (t) atomicAdd(&a.rk_sum[2 * a.W + m], t);
        }
      }
    } else if (act) {
      for (uint32_t q = 0; q < nm; ++q) {
        if (!valid) continue;
        const uint32_t m = member(q);
        const uint32_t wait = sdur(q) - dmin;
        if (wait) atomicAdd(&a.rk_sum[a.W + m], (unsigned long long)wait);
        if (dmin) atomicAdd(&a.rk_sum[2 * a.W + m], (unsigned long long)dmin);
        if (m != last && (unsigned long long)wait > a.wait_margin) x_edge(a, m, last, a.wi ? sit(q) / a.wi : 0, wait);
      }
    }
  }
  flush_link();
  inc = warp_sum_u32(inc); kmis = warp_sum_u32(kmis); pmis = warp_sum_u32(pmis);
  if (lane_id() == 0) {
    if (inc) atomicAdd(&a.cnt->n_incomplete, (unsigned long long)inc);
    if (kmis) atomicAdd(&a.cnt->n_kind_mismatch, (unsigned long long)kmis);
    if (pmis) atomicAdd(&a.cnt->n_payload_mismatch, (unsigned long long)pmis);
  }
}

__global__ void k_cross_big(XArgs a, const uint32_t* big, uint32_t n_big);

static XArgs cross_args(Ctx& c) {
  XArgs a{};
  a.n_xinst = c.n_xinst; a.NCH = c.NCH; a.n_comms = c.n_comms; a.W = c.W; a.xbase = c.xbase.as<uint64_t>();
  a.ch_base = c.ch_base.as<uint64_t>(); a.ch_slot = c.ch_slot.as<uint64_t>(); a.ch_nmin = c.ch_nmin.as<uint32_t>();
  a.coff = c.coff.as<uint64_t>(); a.cmem = c.cmem.as<uint32_t>(); a.ccls = c.ccls.as<uint8_t>();
  a.nsend = c.ch_nsend.as<uint32_t>(); a.nrecv = c.ch_nrecv.as<uint32_t>();
  a.psrc = c.ch_nsend.as<uint32_t>() + c.n_p2p; a.pdst = c.ch_nrecv.as<uint32_t>() + c.n_p2p;
  a.r_nkeys = c.r_nkeys.as<uint32_t>(); a.r_keys = c.r_keys.as<uint32_t>(); a.r_cnt = c.r_cnt.as<uint32_t>();
  a.slots = c.slots.as<uint4>(); a.rec = c.inst_rec.as<uint4>(); a.wait_c = c.wait_c.as<uint32_t>();
  a.lk_key = c.lk_key.as<unsigned long long>(); a.p2p_inst0 = c.p2p_inst0;
  a.nbc_off = c.nbc_off.as<uint64_t>(); a.nbc = c.nbc.as<uint32_t>(); a.nbp = c.nbp.as<uint32_t>(); a.nbp_n = c.nbp_n.as<uint32_t>();
  a.nnz_tot = c.nnz_c + (uint64_t)c.W * PCAP; a.nnz_c = c.nnz_c;
  a.ew = c.ewc.as<unsigned long long>(); a.rk_sum = c.rk_sum.as<unsigned long long>();
  a.wi = c.dcfg.window_iters; a.wait_margin = (unsigned long long)c.lcfg.wait_margin_ns; a.cnt = c.counters.as<Counters>();
  a.p2p_eslot = c.p2p_eslot.as<uint32_t>(); a.xb_smem = 0; a.xe_off = c.xe_off.as<uint64_t>(); a.xe_col = c.xe_col.as<uint32_t>();
  a.p2p_pos = (stage_active(c) || p2p_defer_on(c)) ? 1 : 0; a.pay = c.d_pay; a.meta = c.d_meta; a.rank_off = c.rank_off.as<uint64_t>();
  return a;
}

int launch_cross_reduce(Ctx& c) {
  XArgs a = cross_args(c);
  if (c.n_xinst == 0) return 0;
  int n = 0;
  if (c.n_p2p) {
    if (c.p2p_eslot.ensure(2 * c.n_p2p * 4) != cudaSuccess) return 0;
    a.p2p_eslot = c.p2p_eslot.as<uint32_t>();
    k_p2p_eslot<<<(unsigned)((c.n_p2p + 255) / 256), 256, 0, c.stream>>>(
        (uint32_t)c.n_p2p, c.ch_nsend.as<uint32_t>() + c.n_p2p, c.ch_nrecv.as<uint32_t>() + c.n_p2p, c.nbc_off.as<uint64_t>(),
        c.nbc.as<uint32_t>(), c.nbp.as<uint32_t>(), c.nbp_n.as<uint32_t>(), c.nnz_c, c.p2p_eslot.as<uint32_t>());
    ++n;
  }
  const size_t xsm = (c.NCH + 1) * 8;
  a.xb_smem = xsm <= 48 * 1024 ? 1 : 0;
  static int sms = 0;
  if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
  // one resident wave (MS_XR_MINB CTAs of 256 threads per SM): each warp walks one contiguous chunk
  unsigned blocks = (unsigned)std::min<uint64_t>((c.n_xinst + 255) / 256, (uint64_t)std::max(sms, 1) * MS_XR_MINB);
  k_cross_reduce<<<blocks, 256, a.xb_smem ? xsm : 0, c.stream>>>(a);
  if (c.n_big) {
    k_cross_big<<<dim3(c.n_big, 32), 256, 0, c.stream>>>(a, c.xbig.as<uint32_t>(), c.n_big);
    ++n;
  }
  return n + 1;
}

// Cross collectives with more than XBIG members (e.g. a model-parallel group of TP*PP ranks): one
// CTA per such communicator, one warp per instance, lanes over the members -- the same decisions
// as k_cross_reduce, whose member loop would otherwise run serially in a single warp per instance.
__global__ void __launch_bounds__(256) k_cross_big(XArgs a, const uint32_t* big, uint32_t n_big) {
  if (*((volatile unsigned*)&a.cnt->overflow) & NOT_SPMD) return;
  const uint32_t ch = big[blockIdx.x];
  const uint32_t lane = lane_id(), nw = (blockDim.x >> 5) * gridDim.y;
  const uint32_t wid = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);  // gridDim.y CTAs share a communicator
  const uint32_t nm = (uint32_t)(a.coff[ch + 1] - a.coff[ch]);
  const uint32_t* mem = a.cmem + a.coff[ch];
  const uint32_t nk = (uint32_t)(a.xbase[ch + 1] - a.xbase[ch]), nmin = a.ch_nmin[ch];
  uint32_t inc = 0, kmis = 0;
  for (uint32_t k = wid; k < nk; k += nw) {
    const uint64_t i = a.ch_base[ch] + k, sb = a.ch_slot[ch] + (uint64_t)k * nm;
    const bool complete = k < nmin;
    uint32_t flags = 0, dmin = 0, dmax = 0, last = NONE32;
    bool valid = false;
    if (complete) {
      flags |= SCAN_F_COMPLETE;
      const uint32_t k0 = slot_kind(a.slots[sb].z);
      bool kok = true;
      for (uint32_t q = lane; q < nm; q += 32) kok &= slot_kind(a.slots[sb + q].z) == k0;
      kok = __all_sync(0xFFFFFFFFu, kok);
      if (kok) flags |= SCAN_F_KIND_OK; else ++kmis;
      flags |= SCAN_F_PAYLOAD_OK;  // collectives carry no payload check
      if (kok) {
        valid = true;
        flags |= SCAN_F_VALID;
        uint32_t mn = NONE32, mx = 0;
        for (uint32_t q = lane; q < nm; q += 32) { const uint32_t d = a.slots[sb + q].x; mn = min(mn, d); mx = max(mx, d); }
        for (int o = 16; o > 0; o >>= 1) {
          mn = min(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
          mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
        }
        uint32_t ls = NONE32, nat = 0;  // lowest member with the minimum, tie count
        for (uint32_t q = lane; q < nm; q += 32)
          if (a.slots[sb + q].x == mn) { ls = min(ls, q); ++nat; }
        for (int o = 16; o > 0; o >>= 1) {
          ls = min(ls, __shfl_xor_sync(0xFFFFFFFFu, ls, o));
          nat += __shfl_xor_sync(0xFFFFFFFFu, nat, o);
        }
        dmin = mn; dmax = mx; last = mem[ls];
        if (nat == 1) flags |= SCAN_F_UNIQUE_LAST;
        const uint64_t xo = a.xe_off[ch];
        for (uint32_t q = lane; q < nm; q += 32) {
          const uint32_t m = mem[q];
          const uint4 sq = a.slots[sb + q];
          const uint32_t wait = sq.x - dmin;
          if (wait) atomicAdd(&a.rk_sum[a.W + m], (unsigned long long)wait);
          if (dmin) atomicAdd(&a.rk_sum[2 * a.W + m], (unsigned long long)dmin);
          if (m != last && (unsigned long long)wait > a.wait_margin) {
            const uint32_t win = a.wi ? (sq.z & SLOT_IT_MASK) / a.wi : 0;
            if (xo != ~0ull) atomicAdd(&a.ew[(uint64_t)win * a.nnz_tot + a.xe_col[xo + (uint64_t)q * nm + ls]], (unsigned long long)wait);
            else x_edge(a, m, last, win, wait);
          }
        }
      }
    } else {
      ++inc;  // present members of an incomplete instance wait 0 (k_xwait_scatter)
    }
    if (lane == 0) a.rec[i] = make_uint4(dmin, dmax, last, flags | ((uint32_t)a.ccls[ch] << 8));
    (void)valid;
  }
  if (lane == 0) {
    if (inc) atomicAdd(&a.cnt->n_incomplete, (unsigned long long)inc);
    if (kmis) atomicAdd(&a.cnt->n_kind_mismatch, (unsigned long long)kmis);
  }
}

// Comm-order view of the cross-stage members' waits (COMM_WAIT / EV_WAIT exports): a member's wait is
// its slot's duration minus the instance's dmin (record), scattered to wait_c[comm index of the slot]
// once, on the first export that needs them. A sparse update of the comm-order
// array costs a sector read + write per member, which the analysis itself does not pay.
__global__ void __launch_bounds__(256) k_xwait_scatter(XArgs a) {
  for (uint64_t xi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; xi < a.n_xinst; xi += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t ch = upper_bound_u64(a.xbase, a.NCH + 1, xi) - 1;
    const uint64_t k = xi - a.xbase[ch];
    const bool isp = ch >= a.n_comms;
    const uint32_t nm = isp ? 2u : (uint32_t)(a.coff[ch + 1] - a.coff[ch]);
    const uint64_t sb = a.ch_slot[ch] + k * nm;
    const bool complete = k < a.ch_nmin[ch];
    const uint4 rc = a.rec[a.ch_base[ch] + k];
    for (uint32_t q = 0; q < nm; ++q) {
      bool present = complete;
      if (!present) {
        if (isp) {
          present = (q == 0 ? a.nsend[ch - a.n_comms] : a.nrecv[ch - a.n_comms]) > k;
        } else {
          const uint32_t m = a.cmem[a.coff[ch] + q];
          const uint32_t C = a.r_nkeys[m];
          const uint32_t p = lower_bound_u32(a.r_keys + (uint64_t)m * RCAP, C, (uint32_t)ch);
          present = p < C && a.r_keys[(uint64_t)m * RCAP + p] == (uint32_t)ch && a.r_cnt[(uint64_t)m * RCAP + p] > k;
        }
      }
      if (present) {  // wait = duration - dmin of a valid instance, else 0
        const uint4 sq = a.slots[sb + q];
        a.wait_c[sq.y] = (rc.w & SCAN_F_VALID) ? sq.x - rc.x : 0u;
      }
    }
  }
}

int launch_xwait_scatter(Ctx& c) {
  if (c.n_xinst == 0) return 0;
  XArgs a = cross_args(c);
  unsigned blocks = (unsigned)std::min<uint64_t>((c.n_xinst + 255) / 256, 148ull * 8);
  k_xwait_scatter<<<blocks, 256, 0, c.stream>>>(a);
  return 1;
}

// ----------------------------------------------------------------------------- deferred stage 2
// The first comm position of a tile whose preceding compute segment starts in an earlier tile:
// pslow from the global slow bits (complete after k_fused), late flags from dlate.
__device__ __forceinline__ void k_deferred_row(uint32_t tile, uint32_t row, uint32_t r, uint32_t R, int W, uint4 d4,
                                               const uint32_t* dlate, const uint64_t* bits_off, const uint32_t* bits,
                                               uint32_t* wl_joined, uint32_t* wl_late) {
  const uint32_t di[4] = {d4.x, d4.y, d4.z, d4.w};
  const uint32_t* b = bits + bits_off[r];
  const uint32_t lo = di[1], hi = di[0];
  bool any = false;
  if (lo < hi) {
    const uint32_t w0 = lo >> 5, w1 = (hi - 1) >> 5;
    for (uint32_t w = w0; w <= w1 && !any; ++w) {
      uint32_t m = b[w];
      if (w == w0) m &= 0xFFFFFFFFu << (lo & 31);
      if (w == w1) m &= 0xFFFFFFFFu >> (31 - ((hi - 1) & 31));
      any = m != 0;
    }
  }
  if (!any) return;
  const uint32_t win = di[2];
  atomicAdd(&wl_joined[(uint64_t)win * W + r], 1u);
  if ((dlate[(uint64_t)tile * ((R + 31) / 32) + row / 32] >> (row & 31)) & 1u) atomicAdd(&wl_late[(uint64_t)win * W + r], 1u);
}

// one CTA per tile (most tiles have no deferred position and leave at once), threads over its rows
__global__ void __launch_bounds__(128) k_deferred(uint32_t R, int W, const uint8_t* tile_stage, const uint32_t* dinfo,
                                                  const uint32_t* dlate, const uint64_t* bits_off, const uint32_t* bits,
                                                  uint32_t classes, uint32_t* wl_joined, uint32_t* wl_late, const Counters* cnt) {
  const uint32_t tile = blockIdx.x;
  const uint4 d4 = reinterpret_cast<const uint4*>(dinfo)[tile];
  if (!(d4.w & 1u)) return;
  const uint32_t cls = d4.w >> 8;
  if (!((classes >> (cls - 1)) & 1u)) return;
  if (*((volatile const unsigned*)&cnt->overflow) & NOT_SPMD) return;
  const uint32_t s = tile_stage[tile];
  for (uint32_t row = threadIdx.x; row < R; row += blockDim.x) k_deferred_row(tile, row, s * R + row, R, W, d4, dlate,
                                                                               bits_off, bits, wl_joined, wl_late);
}

int launch_deferred(Ctx& c) {
  if (c.lcfg.stage2_mode != 0 || stage_active(c)) return 0;  // k_stage carries the segments itself
  k_deferred<<<c.n_ftiles, 128, 0, c.stream>>>(
      c.FR, c.W, c.tile_stage.as<uint8_t>(), c.dinfo.as<uint32_t>(), c.dlate.as<uint32_t>(),
      c.r_bits_off.as<uint64_t>(), c.bits.as<uint32_t>(), c.lcfg.stage2_classes, c.wl_joined.as<uint32_t>(),
      c.wl_late.as<uint32_t>(), c.counters.as<Counters>());
  return 1;
}

}  // namespace ms

namespace ms {
// Stage-1 verdict inputs per (window, rank) from the counters k_fused accumulated.
__global__ void k_wd_finish(uint64_t items, const uint32_t* wd_total, const uint32_t* wd_slow, uint8_t* wd_cand,
                            double* wd_frac, uint32_t cand_num, uint32_t cand_den, uint32_t min_samples, Counters* cnt) {
  const uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= items) return;
  const uint32_t total = wd_total[it], slow = wd_slow[it];
  const bool cand = total >= min_samples && (unsigned long long)cand_den * slow > (unsigned long long)cand_num * total;
  wd_cand[it] = cand ? 1 : 0;
  wd_frac[it] = total ? (double)slow / (double)total : 0.0;
  if (total) atomicAdd(&cnt->n_compared, (unsigned long long)total);
  if (slow) atomicAdd(&cnt->n_slow, (unsigned long long)slow);
  if (cand) atomicAdd(&cnt->n_candidates, 1ull);
}

int launch_wd_finish(Ctx& c) {
  const uint64_t items = (uint64_t)c.NW * c.W;
  k_wd_finish<<<(unsigned)((items + 255) / 256), 256, 0, c.stream>>>(items, c.wd_total.as<uint32_t>(), c.wd_slow.as<uint32_t>(),
                                                                     c.wd_cand.as<uint8_t>(), c.wd_frac.as<double>(),
                                                                     c.dcfg.cand_num, c.dcfg.cand_den, c.dcfg.min_samples,
                                                                     c.counters.as<Counters>());
  return 1;
}
}  // namespace ms
