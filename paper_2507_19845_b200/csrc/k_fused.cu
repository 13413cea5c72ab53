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
#include "internal.cuh"

namespace ms {

enum { TY_COMPUTE = 0, TY_TP = 1, TY_DP = 2, TY_XCOLL = 3, TY_P2P = 4 };
constexpr uint32_t NOT_SPMD = 32u;  // Counters.overflow bit: fused path not applicable

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
// One warp per fused tile reads the template rank's row only (1/R of the data): role counts,
// compute / comm / iter_end counts, compute count before the last comm position.
struct PreArgs {
  const uint16_t* kind; const uint32_t* comm; const uint64_t* rank_off; int W, PP;
  uint32_t T, R, n_ftiles; const uint32_t* st_tile0; const uint32_t* st_npos;
  const uint32_t* role_comm; const uint32_t* ncroles;
  uint32_t* cols; Counters* cnt;
};

__global__ void __launch_bounds__(256) k_fused_prepass(PreArgs a) {
  __shared__ uint32_t rcnt[8][ROLES];
  const uint32_t wid = threadIdx.x >> 5, lane = lane_id();
  const uint32_t tile = blockIdx.x * 8 + wid;
  rcnt[wid][lane] = 0;
  __syncwarp();
  if (tile >= a.n_ftiles) return;
  uint32_t s = 0;
  while (s + 1 < (uint32_t)a.PP && a.st_tile0[s + 1] <= tile) ++s;
  const uint32_t p0 = (tile - a.st_tile0[s]) * a.T;
  const uint32_t np = min(a.T, a.st_npos[s] - p0);
  const uint32_t r0 = s * a.R;
  const uint64_t g0 = a.rank_off[r0] + p0;
  const uint32_t* rc = a.role_comm + (uint64_t)r0 * CROLES;
  const uint32_t ncr = a.ncroles[s];
  uint32_t ncomp = 0, ncomm = 0, niter = 0;
  int32_t lastc = -1;
  bool bad = false;
  for (uint32_t q = lane; q < np; q += 32) {
    const uint16_t ko = a.kind[g0 + q];
    const uint32_t kind = ko & 7u;
    niter += (ko >> 3) & 1u;
    if (kind == 0) { ++ncomp; continue; }
    const int role = role_of(kind, a.comm[g0 + q], r0, rc, ncr, a.R, a.W);
    if (role < 0) { bad = true; continue; }
    ++ncomm;
    atomicAdd(&rcnt[wid][role], 1u);
    lastc = (int32_t)q;
  }
  ncomp = warp_sum_u32(ncomp); ncomm = warp_sum_u32(ncomm); niter = warp_sum_u32(niter);
  const int32_t lq = (int32_t)__reduce_max_sync(0xFFFFFFFFu, (unsigned)(lastc + 1)) - 1;
  if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(&a.cnt->overflow, NOT_SPMD);
  __syncwarp();
  const uint64_t n = a.n_ftiles;
  a.cols[(uint64_t)lane * n + tile] = rcnt[wid][lane];
  if (lane == 0) {
    a.cols[(uint64_t)(ROLES + 0) * n + tile] = ncomp;
    a.cols[(uint64_t)(ROLES + 1) * n + tile] = ncomm;
    a.cols[(uint64_t)(ROLES + 2) * n + tile] = niter;
    // compute positions before the last comm position (cc_last), or 0xFFFFFFFF
    a.cols[(uint64_t)(ROLES + 3) * n + tile] = lq >= 0 ? (uint32_t)lq - (ncomm - 1) : NONE32;
  }
}

// F0b: per (stage, column) exclusive scans over the stage's tiles; stage totals. The compute
// column also yields jprev (compute index of the last comm event before the tile).
constexpr int SC_NT = 1024;
__global__ void __launch_bounds__(SC_NT) k_fused_scan(uint32_t n_ftiles, const uint32_t* st_tile0, const uint32_t* cols,
                                                      uint32_t* base, uint32_t* st_tot) {
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
      const uint32_t cc = cols[(uint64_t)(ROLES + 3) * n + t];
      if (cc != NONE32) run = max(run, (int32_t)(base[(uint64_t)ROLES * n + t] + cc));
    }
  }
}

int launch_fused_prepass(Ctx& c) {
  PreArgs a{c.d_kind, c.d_comm, c.rank_off.as<uint64_t>(), c.W, c.PP, c.FT, c.FR, c.n_ftiles, c.st_tile0.as<uint32_t>(),
            c.st_npos.as<uint32_t>(), c.role_comm.as<uint32_t>(), c.ncroles.as<uint32_t>(), c.ft_cols.as<uint32_t>(),
            c.counters.as<Counters>()};
  k_fused_prepass<<<(c.n_ftiles + 7) / 8, 256, 0, c.stream>>>(a);
  k_fused_scan<<<dim3(c.PP, ROLES + 3), SC_NT, 0, c.stream>>>(c.n_ftiles, c.st_tile0.as<uint32_t>(), c.ft_cols.as<uint32_t>(),
                                                              c.ft_base.as<uint32_t>(), c.st_tot.as<uint32_t>());
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
  atomicMax(&a.cnt->max_niter, niter);
  atomicMax(&a.cnt->max_ncomp, ncomp);
  const uint64_t e1 = a.rank_off[r + 1];
  if (e1 > a.rank_off[r]) atomicMax(&a.cnt->n_iters, niter - ((a.kind[e1 - 1] & 8u) ? 1u : 0u) + 1u);
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
struct FusedArgs {
  const uint32_t* dur; const uint16_t* kind; const uint16_t* meta; const uint32_t* comm; const uint32_t* pay;
  const uint64_t* rank_off; int TP, DP, PP, W; uint32_t n_comms; uint32_t T, R, n_ftiles; bool aligned;
  const uint32_t* st_tile0; const uint32_t* st_npos; const uint32_t* ft_base;
  const uint32_t* role_comm; const uint32_t* role_slot; const uint8_t* role_type; const uint32_t* ncroles;
  const uint64_t* coff;
  const uint64_t* ch_base; const uint64_t* ch_slot; const uint32_t* bitmap; const uint32_t* bitpre;
  const uint64_t* comm_off; const uint64_t* comp_off; const uint64_t* bits_off;
  uint32_t* inst_c; uint32_t* wait_c; uint32_t* bits; uint32_t* cref; uint4* rec;
  uint32_t* sdur; uint8_t* skind; uint32_t* sci; uint32_t* sit; uint32_t* p2p_pay; uint8_t* p2p_warm; uint32_t* p2p_iter;
  uint64_t p2p_slot0, p2p_inst0;
  uint32_t* citer; uint32_t NIT1;
  const uint64_t* nbc_off; const uint32_t* nbc; const uint32_t* nbp; const uint32_t* nbp_n; uint64_t nnz_tot, nnz_c;
  unsigned long long* ew; unsigned long long* rk_sum; uint32_t* wl_joined; uint32_t* wl_late;
  uint32_t* dlate; uint32_t* dinfo;
  uint32_t slow_num, slow_den; unsigned long long slow_margin;
  uint32_t wi, classes, mode; unsigned long long late_margin, wait_margin; int want_ref;
  Counters* cnt;
};

constexpr int F_NT = 256;

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

template <int P>
__global__ void __launch_bounds__(F_NT) k_fused(FusedArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const uint32_t T = a.T, R = a.R, TP = (uint32_t)a.TP, DP = (uint32_t)a.DP;
  const uint32_t T1 = T + 1;
  const uint32_t SW = T / 32 + 2;
  // ---- shared memory carve-up
  uint32_t* sd = (uint32_t*)smem_raw;                       // R x (T+1) durations
  uint32_t* sbits = sd + (uint64_t)R * T1;                  // R x SW slow bits
  unsigned long long* rsum = (unsigned long long*)(sbits + (uint64_t)R * SW + ((R * T1 + R * SW) & 1));  // R x 2
  unsigned long long* gsum = rsum + 2 * R;                  // DP (TP groups) + TP (DP groups)
  uint32_t* sjoin = (uint32_t*)(gsum + DP + TP);            // R
  uint32_t* slate = sjoin + R;                              // R
  uint32_t* pk = slate + R;                                 // T
  uint32_t* pj = pk + T;
  uint32_t* pm = pj + T;
  uint32_t* pit = pm + T;
  uint32_t* pjp = pit + T;
  uint32_t* tc = pjp + T;                                   // template comm
  uint16_t* tk = (uint16_t*)(tc + T);                       // template kind_op
  uint16_t* lst = tk + T;                                   // position lists (4 x T)
  uint8_t* ptype = (uint8_t*)(lst + 4 * T);
  uint8_t* prole = ptype + T;
  __shared__ uint32_t rcnt[33][ROLES];
  __shared__ uint32_t scan_sm[33];
  __shared__ int32_t scan_smi[33];
  __shared__ uint32_t nlist[5];
  __shared__ int32_t dpos;
  __shared__ uint32_t bad;

  const uint32_t tile = blockIdx.x;
  uint32_t s = 0;
  while (s + 1 < (uint32_t)a.PP && a.st_tile0[s + 1] <= tile) ++s;
  const uint32_t p0 = (tile - a.st_tile0[s]) * T;
  const uint32_t np = min(T, a.st_npos[s] - p0);
  const uint32_t sbase = s * R;
  const uint64_t n = a.n_ftiles;
  const uint32_t j0 = a.ft_base[(uint64_t)ROLES * n + tile];
  const uint32_t m0 = a.ft_base[(uint64_t)(ROLES + 1) * n + tile];
  const uint32_t it0 = a.ft_base[(uint64_t)(ROLES + 2) * n + tile];
  const uint32_t jp0 = a.ft_base[(uint64_t)(ROLES + 3) * n + tile];
  const uint32_t wb = j0 >> 5;
  const uint32_t w_tile = a.wi ? it0 / a.wi : 0;
  const uint32_t tid = threadIdx.x;
  const uint32_t ncr = a.ncroles[s];
  const uint32_t* rc0 = a.role_comm + (uint64_t)sbase * CROLES;

  // ---- (1) template row + shared-memory init
  if (tid < 5) nlist[tid] = 0;
  if (tid == 0) { dpos = -1; bad = 0; }
  for (uint32_t i = tid; i < R * SW; i += F_NT) sbits[i] = 0;
  for (uint32_t i = tid; i < R; i += F_NT) { rsum[2 * i] = 0; rsum[2 * i + 1] = 0; sjoin[i] = 0; slate[i] = 0; }
  for (uint32_t i = tid; i < DP + TP; i += F_NT) gsum[i] = 0;
  for (uint32_t i = tid; i < 33 * ROLES; i += F_NT) (&rcnt[0][0])[i] = 0;
  const uint64_t g0 = a.rank_off[sbase] + p0;
  for (uint32_t p = tid; p < T; p += F_NT) {
    if (p < np) { tk[p] = a.kind[g0 + p]; tc[p] = a.comm[g0 + p]; }
    else { tk[p] = 0; tc[p] = 0; }
  }
  __syncthreads();
  // ---- (2) per-position info from the template row: type, role, j, m, iteration, k, jprev
  const uint32_t PPT = (T + F_NT - 1) / F_NT;
  uint32_t lc = 0, lm = 0, li = 0;
  for (uint32_t q = 0; q < PPT; ++q) {
    const uint32_t p = tid * PPT + q;
    if (p >= np) break;
    const uint32_t kind = tk[p] & 7u;
    int role = -1;
    uint8_t ty = TY_COMPUTE;
    if (kind) {
      role = role_of(kind, tc[p], sbase, rc0, ncr, R, a.W);
      if (role < 0) { bad = 1; role = 0; }
      ty = role >= 16 ? (uint8_t)TY_P2P : a.role_type[s * ROLES + role];
      ++lm;
    } else {
      ++lc;
    }
    ptype[p] = ty; prole[p] = (uint8_t)(role < 0 ? 255 : role);
    li += (tk[p] >> 3) & 1u;
  }
  uint32_t tc_, tm_, ti_;
  uint32_t ec = block_excl_sum<F_NT>(lc, tc_, scan_sm);
  uint32_t em = block_excl_sum<F_NT>(lm, tm_, scan_sm);
  uint32_t ei = block_excl_sum<F_NT>(li, ti_, scan_sm);
  int32_t mylastj = -1;
  for (uint32_t q = 0; q < PPT; ++q) {
    const uint32_t p = tid * PPT + q;
    if (p >= np) break;
    pj[p] = j0 + ec; pm[p] = m0 + em; pit[p] = it0 + ei;
    const bool isc = (tk[p] & 7u) == 0;
    if (!isc) mylastj = (int32_t)(j0 + ec);
    ec += isc; em += !isc; ei += (tk[p] >> 3) & 1u;
  }
  // jprev: compute index of the previous comm position (or the tile base)
  int32_t totj;
  int32_t exj = block_excl_max<F_NT>(mylastj, totj, scan_smi);
  int32_t run = max((int32_t)jp0, exj);
  for (uint32_t q = 0; q < PPT; ++q) {
    const uint32_t p = tid * PPT + q;
    if (p >= np) break;
    if (tk[p] & 7u) { pjp[p] = (uint32_t)run; run = (int32_t)pj[p]; }
  }
  // in-tile occurrence rank per role (warp-chunked match) + lists
  for (uint32_t ch = tid >> 5; ch * 32 < T; ch += F_NT / 32) {
    const uint32_t p = ch * 32 + lane_id();
    const bool in = p < np && (tk[p] & 7u);
    const uint32_t role = in ? prole[p] : 0xFFFFu;
    const unsigned act = __ballot_sync(0xFFFFFFFFu, in);
    const unsigned mm = __match_any_sync(0xFFFFFFFFu, role);
    if (in) {
      const unsigned grp = mm & act;
      pk[p] = __popc(grp & ((1u << lane_id()) - 1u));
      if (lane_id() == (uint32_t)(__ffs(grp) - 1)) rcnt[ch][role] = __popc(grp);
    }
    if (p < np) {
      const uint8_t ty = ptype[p];
      const uint32_t li_ = (tk[p] & 7u) == 0 ? 0u : (ty == TY_TP ? 1u : (ty == TY_DP ? 2u : 3u));
      const uint32_t slot = atomicAdd(&nlist[li_], 1u);
      lst[li_ * T + slot] = (uint16_t)p;
      if ((tk[p] >> 3) & 1u) { const uint32_t sl = atomicAdd(&nlist[4], 1u); (void)sl; }
    }
  }
  __syncthreads();
  if (tid < ROLES) {
    uint32_t acc = a.ft_base[(uint64_t)tid * n + tile];
    for (uint32_t ch = 0; ch * 32 < T; ++ch) { const uint32_t v = rcnt[ch][tid]; rcnt[ch][tid] = acc; acc += v; }
  }
  __syncthreads();
  for (uint32_t p = tid; p < np; p += F_NT)
    if (tk[p] & 7u) pk[p] += rcnt[p >> 5][prole[p]];
  if (tid == 0 && a.mode == 0) {
    // the first comm position of the tile reaches back across the tile start: defer its stage-2
    for (uint32_t p = 0; p < np; ++p)
      if (tk[p] & 7u) {
        if ((ptype[p] == TY_TP || ptype[p] == TY_DP) && pjp[p] < j0) dpos = (int32_t)p;
        break;
      }
  }
  // ---- (3) stream every rank row of the tile: verify against the template, stage durations
  for (uint32_t wq = tid >> 5; wq < R * ((T + 127) / 128); wq += F_NT / 32) {
    const uint32_t row = wq / ((T + 127) / 128), chunk = wq % ((T + 127) / 128);
    const uint32_t r = sbase + row;
    const uint32_t pb = chunk * 128 + lane_id() * 4;
    const uint64_t g = a.rank_off[r] + p0 + pb;
    uint16_t ko[4]; uint32_t cm[4], du[4];
    if (a.aligned && pb + 4 <= np) {
      const uint2 kv = __ldg(reinterpret_cast<const uint2*>(a.kind + g));
      const uint4 cv = __ldg(reinterpret_cast<const uint4*>(a.comm + g));
      const uint4 dv = __ldg(reinterpret_cast<const uint4*>(a.dur + g));
      ko[0] = (uint16_t)kv.x; ko[1] = (uint16_t)(kv.x >> 16); ko[2] = (uint16_t)kv.y; ko[3] = (uint16_t)(kv.y >> 16);
      cm[0] = cv.x; cm[1] = cv.y; cm[2] = cv.z; cm[3] = cv.w;
      du[0] = dv.x; du[1] = dv.y; du[2] = dv.z; du[3] = dv.w;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const bool v = pb + i < np;
        ko[i] = v ? a.kind[g + i] : 0; cm[i] = v ? a.comm[g + i] : 0; du[i] = v ? a.dur[g + i] : 0;
      }
    }
    unsigned long long scomp = 0, sinb = 0;
    bool mis = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t p = pb + i;
      if (p >= np) break;
      if (ko[i] != tk[p]) mis = true;
      const uint8_t ty = ptype[p];
      const uint32_t role = prole[p];
      if ((tk[p] & 7u) == 0) {
        scomp += du[i];
      } else if (role < 16) {
        if (cm[i] != a.role_comm[(uint64_t)r * CROLES + role]) mis = true;
        if (ty == TY_TP || ty == TY_DP) sinb += du[i];
      } else {
        const int ds = (int)(role & 7u) - 4;
        if ((int)cm[i] != (int)r + ds * (int)R) mis = true;
      }
      sd[row * T1 + p] = du[i];
    }
    if (__any_sync(0xFFFFFFFFu, mis) && lane_id() == 0) bad = 1;
    scomp = warp_sum_u64(scomp); sinb = warp_sum_u64(sinb);
    if (lane_id() == 0) {
      if (scomp) atomicAdd(&rsum[2 * row], scomp);
      if (sinb) atomicAdd(&rsum[2 * row + 1], sinb);
    }
  }
  __syncthreads();
  if (bad) { if (tid == 0) atomicOr(&a.cnt->overflow, NOT_SPMD); return; }
  // ---- (4) phase A: stage 1 on every compute position (LOO lower median over the DP peers)
  const uint32_t nc = nlist[0];
  if (P >= 2) {
    const int q = ((int)DP - 2) / 2;
    for (uint32_t it = tid; it < nc * TP; it += F_NT) {
      const uint32_t p = lst[it / TP], tp = it % TP;
      // pad to P with L low (0) and P-DP-L high (max) sentinels so that the two order statistics
      // needed, s[q] and s[q+1] with q = floor((DP-2)/2), land at the fixed indices P/2-1, P/2
      const int L = P / 2 - 1 - q;
      uint32_t x[P], v[P];
#pragma unroll
      for (int d = 0; d < P; ++d) {
        x[d] = d < (int)DP ? sd[(tp + TP * d) * T1 + p] : 0xFFFFFFFFu;
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
      const uint32_t j = pj[p];
#pragma unroll
      for (int d = 0; d < P; ++d) {
        if (d < (int)DP) {
          const uint32_t ref = x[d] > va ? va : vb;
          const unsigned long long du = x[d];
          const bool slow = (unsigned long long)a.slow_den * du > (unsigned long long)a.slow_num * ref &&
                            du > (unsigned long long)ref + a.slow_margin;
          const uint32_t row = tp + TP * d;
          if (slow) atomicOr(&sbits[row * SW + (j >> 5) - wb], 1u << (j & 31));
          if (a.want_ref) a.cref[a.comp_off[sbase + row] + j] = ref;
        }
      }
    }
  }
  // iteration boundaries (compute index at which the next iteration starts), for every rank
  for (uint32_t p = tid; p < np; p += F_NT) {
    if (!((tk[p] >> 3) & 1u)) continue;
    const uint32_t v = pj[p] + ((tk[p] & 7u) == 0 ? 1u : 0u);
    for (uint32_t row = 0; row < R; ++row) a.citer[(uint64_t)(sbase + row) * a.NIT1 + pit[p] + 1] = v;
  }
  __syncthreads();
  // ---- (5) phase B: TP / DP instances (all members in the tile) and cross-stage scatters
  const uint32_t ntp = nlist[1], ndp = nlist[2], nx = nlist[3];
  const uint32_t I1 = ntp * DP, I2 = I1 + ndp * TP, I3 = I2 + nx * R;
  for (uint32_t it = tid; it < I3; it += F_NT) {
    if (it < I2) {
      const bool istp = it < I1;
      const uint32_t p = istp ? lst[T + it / DP] : lst[2 * T + (it - I1) / TP];
      const uint32_t g = istp ? it % DP : (it - I1) % TP;
      const uint32_t nm = istp ? TP : DP, stride = istp ? 1u : TP, row0 = istp ? TP * g : g;
      const uint32_t role = prole[p];
      const uint32_t cid = a.role_comm[(uint64_t)(sbase + row0) * CROLES + role];
      const uint64_t inst = a.ch_base[cid] + pk[p];
      uint32_t dmin = 0xFFFFFFFFu, dmax = 0, ls = 0, nat = 0;
      for (uint32_t q = 0; q < nm; ++q) {
        const uint32_t d = sd[(row0 + q * stride) * T1 + p];
        if (d < dmin) { dmin = d; ls = q; nat = 1; } else if (d == dmin) ++nat;
        dmax = max(dmax, d);
      }
      const uint32_t cls = istp ? 1u : 2u;
      const uint32_t last = sbase + row0 + ls * stride;
      a.rec[inst] = make_uint4(dmin, dmax, last, (SCAN_F_COMPLETE | SCAN_F_KIND_OK | SCAN_F_PAYLOAD_OK | SCAN_F_VALID |
                                                  (nat == 1 ? SCAN_F_UNIQUE_LAST : 0u)) | (cls << 8));
      atomicAdd(&gsum[istp ? g : DP + g], (unsigned long long)dmin);
      const uint32_t win = a.wi ? pit[p] / a.wi : 0;
      const bool elig = (a.classes >> (cls - 1)) & 1u;
      const bool late_ok = nat == 1 && (unsigned long long)(dmax - dmin) > a.late_margin;
      for (uint32_t q = 0; q < nm; ++q) {
        const uint32_t row = row0 + q * stride, r = sbase + row;
        const uint32_t d = sd[row * T1 + p];
        const uint64_t ci = a.comm_off[r] + pm[p];
        a.inst_c[ci] = (uint32_t)inst;
        const uint32_t wait = d - dmin;
        a.wait_c[ci] = wait;
        if (q != ls && (unsigned long long)wait > a.wait_margin) add_edge(a, r, last, win, wait);
        if (!elig) continue;
        const bool lt = q == ls && late_ok;
        if ((int32_t)p == dpos) {
          if (lt) atomicOr(&a.dlate[(uint64_t)tile * ((R + 31) / 32) + row / 32], 1u << (row & 31));
          continue;
        }
        const bool pslow = a.mode ? true : sbits_any(sbits + row * SW, wb, pjp[p], pj[p]);
        if (!pslow) continue;
        if (win == w_tile) { atomicAdd(&sjoin[row], 1u); if (lt) atomicAdd(&slate[row], 1u); }
        else { atomicAdd(&a.wl_joined[(uint64_t)win * a.W + r], 1u); if (lt) atomicAdd(&a.wl_late[(uint64_t)win * a.W + r], 1u); }
      }
    } else {
      const uint32_t x = it - I2;
      const uint32_t p = lst[3 * T + x / R], row = x % R, r = sbase + row;
      const uint32_t role = prole[p];
      const uint64_t e = a.rank_off[r] + p0 + p;
      uint64_t ch; uint32_t nm, slot;
      bool send = false;
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
      const uint64_t inst = a.ch_base[ch] + pk[p];
      const uint64_t si = a.ch_slot[ch] + (uint64_t)pk[p] * nm + slot;
      const uint64_t ci = a.comm_off[r] + pm[p];
      a.inst_c[ci] = (uint32_t)inst;
      a.sdur[si] = sd[row * T1 + p];
      a.skind[si] = (uint8_t)(tk[p] & 7u);
      a.sci[si] = (uint32_t)ci;
      a.sit[si] = pit[p];
      if (role >= 16) {
        a.p2p_pay[si - a.p2p_slot0] = a.pay[e];
        if (send) {
          a.p2p_warm[inst - a.p2p_inst0] = (uint8_t)((a.meta[e] >> 14) & 1u);
          a.p2p_iter[inst - a.p2p_inst0] = pit[p];
        }
      }
    }
  }
  __syncthreads();
  // ---- (6) flush: slow bits, per-rank sums, stage-2 counters, deferred position
  const uint32_t nct = nlist[0];
  if (nct) {
    const uint32_t w_first = j0 >> 5, w_last = (j0 + nct - 1) >> 5;
    const uint32_t nw = w_last - w_first + 1;
    for (uint32_t i = tid; i < R * nw; i += F_NT) {
      const uint32_t row = i / nw, w = w_first + i % nw;
      const uint32_t v = sbits[row * SW + (w - wb)];
      if (v) atomicOr(&a.bits[a.bits_off[sbase + row] + w], v);
    }
  }
  for (uint32_t row = tid; row < R; row += F_NT) {
    const uint32_t r = sbase + row;
    const unsigned long long tr = gsum[row / TP] + gsum[DP + row % TP];
    if (rsum[2 * row]) atomicAdd(&a.rk_sum[r], rsum[2 * row]);
    if (rsum[2 * row + 1] - tr) atomicAdd(&a.rk_sum[a.W + r], rsum[2 * row + 1] - tr);
    if (tr) atomicAdd(&a.rk_sum[2 * a.W + r], tr);
    if (sjoin[row]) atomicAdd(&a.wl_joined[(uint64_t)w_tile * a.W + r], sjoin[row]);
    if (slate[row]) atomicAdd(&a.wl_late[(uint64_t)w_tile * a.W + r], slate[row]);
  }
  if (tid == 0) {
    uint32_t* di = a.dinfo + (uint64_t)tile * 4;
    if (dpos >= 0) {
      const uint32_t p = (uint32_t)dpos;
      di[0] = pj[p]; di[1] = pjp[p]; di[2] = a.wi ? pit[p] / a.wi : 0; di[3] = 1u | ((uint32_t)ptype[p] << 8);
    } else {
      di[3] = 0;
    }
  }
}

size_t fused_smem_bytes(uint32_t T, uint32_t R, uint32_t TP, uint32_t DP) {
  const uint32_t SW = T / 32 + 2;
  size_t b = (size_t)R * (T + 1) * 4 + (size_t)R * SW * 4 + 4 /*align*/ + (size_t)R * 16 + (size_t)(DP + TP) * 8 +
             (size_t)R * 8 + (size_t)T * 4 * 6 + (size_t)T * 2 + (size_t)T * 2 * 4 + (size_t)T * 2;
  return (b + 15) & ~size_t(15);
}

int launch_fused(Ctx& c) {
  FusedArgs a;
  a.dur = c.d_dur; a.kind = c.d_kind; a.meta = c.d_meta; a.comm = c.d_comm; a.pay = c.d_pay;
  a.rank_off = c.rank_off.as<uint64_t>(); a.TP = c.TP; a.DP = c.DP; a.PP = c.PP; a.W = c.W; a.n_comms = c.n_comms;
  a.T = c.FT; a.R = c.FR; a.n_ftiles = c.n_ftiles; a.aligned = c.rows_aligned;
  a.st_tile0 = c.st_tile0.as<uint32_t>(); a.st_npos = c.st_npos.as<uint32_t>(); a.ft_base = c.ft_base.as<uint32_t>();
  a.role_comm = c.role_comm.as<uint32_t>(); a.role_slot = c.role_slot.as<uint32_t>(); a.role_type = c.role_type.as<uint8_t>();
  a.ncroles = c.ncroles.as<uint32_t>(); a.coff = c.coff.as<uint64_t>();
  a.ch_base = c.ch_base.as<uint64_t>(); a.ch_slot = c.ch_slot.as<uint64_t>(); a.bitmap = c.bitmap.as<uint32_t>();
  a.bitpre = c.bitpre.as<uint32_t>(); a.comm_off = c.r_comm_off.as<uint64_t>(); a.comp_off = c.r_comp_off.as<uint64_t>();
  a.bits_off = c.r_bits_off.as<uint64_t>(); a.inst_c = c.inst_c.as<uint32_t>(); a.wait_c = c.wait_c.as<uint32_t>();
  a.bits = c.bits.as<uint32_t>(); a.cref = c.cref.as<uint32_t>(); a.rec = c.inst_rec.as<uint4>();
  a.sdur = c.sdur.as<uint32_t>(); a.skind = c.skind.as<uint8_t>(); a.sci = c.sci.as<uint32_t>(); a.sit = c.sit.as<uint32_t>();
  a.p2p_pay = c.p2p_pay.as<uint32_t>(); a.p2p_warm = c.p2p_warm.as<uint8_t>(); a.p2p_iter = c.p2p_iter.as<uint32_t>();
  a.p2p_slot0 = c.p2p_slot0; a.p2p_inst0 = c.p2p_inst0; a.citer = c.citer.as<uint32_t>(); a.NIT1 = c.NIT + 1;
  a.nbc_off = c.nbc_off.as<uint64_t>(); a.nbc = c.nbc.as<uint32_t>(); a.nbp = c.nbp.as<uint32_t>();
  a.nbp_n = c.nbp_n.as<uint32_t>(); a.nnz_tot = c.nnz_c + (uint64_t)c.W * PCAP; a.nnz_c = c.nnz_c;
  a.ew = c.ewc.as<unsigned long long>(); a.rk_sum = c.rk_sum.as<unsigned long long>();
  a.wl_joined = c.wl_joined.as<uint32_t>(); a.wl_late = c.wl_late.as<uint32_t>();
  a.dlate = c.dlate.as<uint32_t>(); a.dinfo = c.dinfo.as<uint32_t>();
  a.slow_num = c.dcfg.slow_num; a.slow_den = c.dcfg.slow_den; a.slow_margin = c.dcfg.slow_margin_ns;
  a.wi = c.dcfg.window_iters; a.classes = c.lcfg.stage2_classes; a.mode = c.lcfg.stage2_mode;
  a.late_margin = c.lcfg.late_margin_ns; a.wait_margin = c.lcfg.wait_margin_ns; a.want_ref = c.dcfg.want_ref ? 1 : 0;
  a.cnt = c.counters.as<Counters>();
  const size_t sm = fused_smem_bytes(c.FT, c.FR, c.TP, c.DP);
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
  uint64_t n_inst, NCH; uint32_t n_comms; int W;
  const uint64_t* ch_base; const uint64_t* ch_slot; const uint32_t* ch_nmin; const uint64_t* coff; const uint32_t* cmem;
  const uint8_t* ccls; const uint32_t* nsend; const uint32_t* nrecv; const uint32_t* psrc; const uint32_t* pdst;
  const uint32_t* r_nkeys; const uint32_t* r_keys; const uint32_t* r_cnt;
  const uint32_t* sdur; const uint8_t* skind; const uint32_t* sci; const uint32_t* sit; const uint32_t* p2p_pay;
  const uint8_t* p2p_warm; uint64_t p2p_slot0, p2p_inst0;
  uint4* rec; uint32_t* wait_c;
  const uint64_t* nbc_off; const uint32_t* nbc; const uint32_t* nbp; const uint32_t* nbp_n; uint64_t nnz_tot, nnz_c;
  unsigned long long* ew; unsigned long long* rk_sum; uint32_t wi; unsigned long long wait_margin;
  Counters* cnt;
};

__device__ __forceinline__ void x_edge(const XArgs& a, uint32_t r, uint32_t L, uint32_t win, uint32_t wait) {
  const uint64_t nb0 = a.nbc_off[r], nb1 = a.nbc_off[r + 1];
  uint64_t idx;
  const uint32_t pc = lower_bound_u32(a.nbc + nb0, (uint32_t)(nb1 - nb0), L);
  if (pc < nb1 - nb0 && a.nbc[nb0 + pc] == L) idx = nb0 + pc;
  else idx = a.nnz_c + (uint64_t)r * PCAP + lower_bound_u32(a.nbp + (uint64_t)r * PCAP, a.nbp_n[r], L);
  atomicAdd(&a.ew[(uint64_t)win * a.nnz_tot + idx], (unsigned long long)wait);
}

__global__ void __launch_bounds__(256) k_cross_reduce(XArgs a) {
  if (*((volatile unsigned*)&a.cnt->overflow) & NOT_SPMD) return;  // fused results void: general path reruns
  uint32_t inc = 0, kmis = 0, pmis = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n_inst; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t ch = upper_bound_u64(a.ch_base, a.NCH + 1, i) - 1;
    const bool isp = ch >= a.n_comms;
    uint32_t cls = 0, nm = 2;
    if (!isp) {
      cls = a.ccls[ch];
      if (cls == 1 || cls == 2) continue;  // TP / DP group: finished inside k_fused
      nm = (uint32_t)(a.coff[ch + 1] - a.coff[ch]);
    }
    const uint64_t k = i - a.ch_base[ch];
    const uint64_t sb = a.ch_slot[ch] + k * nm;
    uint32_t flags = 0;
    if (isp && a.p2p_warm[i - a.p2p_inst0]) flags |= SCAN_F_WARMUP;
    uint32_t dmin = 0, dmax = 0, last = NONE32;
    auto member = [&](uint32_t q) -> uint32_t {
      return isp ? (q == 0 ? a.psrc[ch - a.n_comms] : a.pdst[ch - a.n_comms]) : a.cmem[a.coff[ch] + q];
    };
    auto present = [&](uint32_t q) -> bool {
      if (isp) return (q == 0 ? a.nsend[ch - a.n_comms] : a.nrecv[ch - a.n_comms]) > k;
      const uint32_t m = a.cmem[a.coff[ch] + q];
      const uint32_t C = a.r_nkeys[m];
      const uint32_t p = lower_bound_u32(a.r_keys + (uint64_t)m * RCAP, C, (uint32_t)ch);
      return p < C && a.r_keys[(uint64_t)m * RCAP + p] == (uint32_t)ch && a.r_cnt[(uint64_t)m * RCAP + p] > k;
    };
    bool valid = false;
    if (k < a.ch_nmin[ch]) {
      flags |= SCAN_F_COMPLETE;
      bool kind_ok = true, pay_ok = true;
      if (!isp) {
        const uint8_t k0 = a.skind[sb];
        for (uint32_t q = 1; q < nm; ++q) if (a.skind[sb + q] != k0) kind_ok = false;
      } else {
        pay_ok = a.p2p_pay[sb - a.p2p_slot0] == a.p2p_pay[sb + 1 - a.p2p_slot0];
      }
      if (kind_ok) flags |= SCAN_F_KIND_OK; else ++kmis;
      if (pay_ok) flags |= SCAN_F_PAYLOAD_OK; else ++pmis;
      if (kind_ok && pay_ok) {
        valid = true;
        flags |= SCAN_F_VALID;
        dmin = NONE32;
        uint32_t ls = 0, nat = 0;
        for (uint32_t q = 0; q < nm; ++q) {
          const uint32_t d = a.sdur[sb + q];
          if (d < dmin) { dmin = d; ls = q; nat = 1; } else if (d == dmin) ++nat;
          dmax = max(dmax, d);
        }
        if (nat == 1) flags |= SCAN_F_UNIQUE_LAST;
        last = member(ls);
      }
    } else {
      ++inc;
    }
    a.rec[i] = make_uint4(dmin, dmax, last, flags | (cls << 8));
    for (uint32_t q = 0; q < nm; ++q) {
      if (!(flags & SCAN_F_COMPLETE) && !present(q)) continue;
      const uint32_t ci = a.sci[sb + q];
      if (!valid) { a.wait_c[ci] = 0; continue; }
      const uint32_t m = member(q);
      const uint32_t wait = a.sdur[sb + q] - dmin;
      a.wait_c[ci] = wait;
      if (wait) atomicAdd(&a.rk_sum[a.W + m], (unsigned long long)wait);
      if (dmin) atomicAdd(&a.rk_sum[2 * a.W + m], (unsigned long long)dmin);
      if (m != last && (unsigned long long)wait > a.wait_margin) x_edge(a, m, last, a.wi ? a.sit[sb + q] / a.wi : 0, wait);
    }
  }
  inc = warp_sum_u32(inc); kmis = warp_sum_u32(kmis); pmis = warp_sum_u32(pmis);
  if (lane_id() == 0) {
    if (inc) atomicAdd(&a.cnt->n_incomplete, (unsigned long long)inc);
    if (kmis) atomicAdd(&a.cnt->n_kind_mismatch, (unsigned long long)kmis);
    if (pmis) atomicAdd(&a.cnt->n_payload_mismatch, (unsigned long long)pmis);
  }
}

int launch_cross_reduce(Ctx& c) {
  if (c.n_inst == 0) return 0;
  XArgs a{c.n_inst, c.NCH, c.n_comms, c.W, c.ch_base.as<uint64_t>(), c.ch_slot.as<uint64_t>(), c.ch_nmin.as<uint32_t>(),
          c.coff.as<uint64_t>(), c.cmem.as<uint32_t>(), c.ccls.as<uint8_t>(), c.ch_nsend.as<uint32_t>(),
          c.ch_nrecv.as<uint32_t>(), c.ch_nsend.as<uint32_t>() + c.n_p2p, c.ch_nrecv.as<uint32_t>() + c.n_p2p,
          c.r_nkeys.as<uint32_t>(), c.r_keys.as<uint32_t>(), c.r_cnt.as<uint32_t>(), c.sdur.as<uint32_t>(),
          c.skind.as<uint8_t>(), c.sci.as<uint32_t>(), c.sit.as<uint32_t>(), c.p2p_pay.as<uint32_t>(),
          c.p2p_warm.as<uint8_t>(), c.p2p_slot0, c.p2p_inst0, c.inst_rec.as<uint4>(), c.wait_c.as<uint32_t>(),
          c.nbc_off.as<uint64_t>(), c.nbc.as<uint32_t>(), c.nbp.as<uint32_t>(), c.nbp_n.as<uint32_t>(),
          c.nnz_c + (uint64_t)c.W * PCAP, c.nnz_c, c.ewc.as<unsigned long long>(), c.rk_sum.as<unsigned long long>(),
          c.dcfg.window_iters, (unsigned long long)c.lcfg.wait_margin_ns, c.counters.as<Counters>()};
  unsigned blocks = (unsigned)std::min<uint64_t>((c.n_inst + 255) / 256, 148ull * 16);
  k_cross_reduce<<<blocks, 256, 0, c.stream>>>(a);
  return 1;
}

// ----------------------------------------------------------------------------- deferred stage 2
// The first comm position of a tile whose preceding compute segment starts in an earlier tile:
// pslow from the global slow bits (complete after k_fused), late flags from dlate.
__global__ void k_deferred(uint32_t n_ftiles, int PP, uint32_t R, int W, const uint32_t* st_tile0, const uint32_t* dinfo,
                           const uint32_t* dlate, const uint64_t* bits_off, const uint32_t* bits, uint32_t classes,
                           uint32_t* wl_joined, uint32_t* wl_late, const Counters* cnt) {
  const uint64_t it = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= (uint64_t)n_ftiles * R) return;
  if (*((volatile const unsigned*)&cnt->overflow) & NOT_SPMD) return;
  const uint32_t tile = (uint32_t)(it / R), row = (uint32_t)(it % R);
  const uint32_t* di = dinfo + (uint64_t)tile * 4;
  if (!(di[3] & 1u)) return;
  const uint32_t cls = di[3] >> 8;
  if (!((classes >> (cls - 1)) & 1u)) return;
  uint32_t s = 0;
  while (s + 1 < (uint32_t)PP && st_tile0[s + 1] <= tile) ++s;
  const uint32_t r = s * R + row;
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

int launch_deferred(Ctx& c) {
  if (c.lcfg.stage2_mode != 0) return 0;
  const uint64_t items = (uint64_t)c.n_ftiles * c.FR;
  k_deferred<<<(unsigned)((items + 255) / 256), 256, 0, c.stream>>>(
      c.n_ftiles, c.PP, c.FR, c.W, c.st_tile0.as<uint32_t>(), c.dinfo.as<uint32_t>(), c.dlate.as<uint32_t>(),
      c.r_bits_off.as<uint64_t>(), c.bits.as<uint32_t>(), c.lcfg.stage2_classes, c.wl_joined.as<uint32_t>(),
      c.wl_late.as<uint32_t>(), c.counters.as<Counters>());
  return 1;
}

}  // namespace ms
