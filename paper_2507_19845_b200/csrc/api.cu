// api.cu — C ABI (include/megascan/scan.h): context, ingest, and the host orchestration of the
// A1-A8 kernels. No CPU fallback: every analysis step runs in the kernels of k_match.cu,
// k_stats.cu; this file only sizes buffers, launches, and reads back counters.
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <numeric>
#include <sstream>
#include "internal.cuh"

#include <cstdlib>

using namespace ms;

void ms::resolve_timing(Ctx& c) {
  for (auto& p : c.pend) {
    float ms_ = 0;
    if (cudaEventElapsedTime(&ms_, p.a, p.b) == cudaSuccess) { c.kms[p.k] += ms_; c.kcnt[p.k] += 1; }
    c.evpool.push_back(p.a); c.evpool.push_back(p.b);
  }
  c.pend.clear();
}


namespace {
constexpr int FILL_MAX = 24;
struct FillArgs { uint8_t* p[FILL_MAX]; uint64_t n[FILL_MAX]; uint32_t v[FILL_MAX]; int k; };
// byte fills of up to FILL_MAX segments: 16-byte stores on the aligned body, bytes at the ends
__global__ void k_fill(FillArgs a) {
  const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, st = (uint64_t)gridDim.x * blockDim.x;
  for (int s = 0; s < a.k; ++s) {
    uint8_t* p = a.p[s];
    const uint64_t n = a.n[s];
    const uint32_t b = a.v[s] & 0xFFu, w = b * 0x01010101u;
    const uint64_t h16 = (16 - ((uintptr_t)p & 15)) & 15, head = n < h16 ? n : h16, nv = (n - head) / 16;
    for (uint64_t i = t0; i < head; i += st) p[i] = (uint8_t)b;
    uint4* q = reinterpret_cast<uint4*>(p + head);
    for (uint64_t i = t0; i < nv; i += st) q[i] = make_uint4(w, w, w, w);
    for (uint64_t i = head + nv * 16 + t0; i < n; i += st) p[i] = (uint8_t)b;
  }
}
}  // namespace

int ms::flush_fills(Ctx& c) {
  for (size_t i = 0; i < c.fills.size(); i += FILL_MAX) {
    FillArgs a{};
    a.k = (int)std::min<size_t>(FILL_MAX, c.fills.size() - i);
    for (int j = 0; j < a.k; ++j) {
      a.p[j] = static_cast<uint8_t*>(c.fills[i + j].p); a.n[j] = c.fills[i + j].n; a.v[j] = c.fills[i + j].v;
    }
    k_fill<<<296, 256, 0, c.stream>>>(a);
    c.launches += 1;
  }
  c.fills.clear();
  return 0;
}

const uint32_t* ms::tile_order_ptr(Ctx& c) {
  static int on = -1;
  if (on < 0) { const char* e = std::getenv("MS_TILE_ORDER"); on = e ? std::atoi(e) : 1; }
  return on ? c.tile_order.as<uint32_t>() : nullptr;
}

scan_status ms::sync_read(Ctx& c) {
  flush_fills(c);
  CK(cudaMemcpyAsync(&c.hc, c.counters.p, sizeof(Counters), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  CK(cudaGetLastError());
  resolve_timing(c);
  return SCAN_OK;
}

namespace {

__global__ void k_citer_fill(int W, uint32_t NIT1, const uint32_t* r_ncomp, uint32_t* citer) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (uint64_t)W * NIT1) return;
  const uint32_t r = (uint32_t)(i / NIT1), q = (uint32_t)(i % NIT1);
  citer[i] = q == 0 ? 0u : r_ncomp[r];
}

}  // namespace

extern "C" {

scan_status scan_create(scan_ctx** out, int cuda_device, void* cuda_stream) {
  if (!out) return SCAN_E_INVALID_ARG;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return SCAN_E_CUDA;
  if (cuda_device < 0 || cuda_device >= n) return SCAN_E_INVALID_ARG;
  if (cudaSetDevice(cuda_device) != cudaSuccess) return SCAN_E_CUDA;
  if (const char* e = std::getenv("MS_L2_FETCH")) {  // experiment: L2 fetch granularity hint (bytes)
    const cudaError_t le = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)std::atoi(e));
    size_t v = 0;
    cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    std::fprintf(stderr, "[MS_L2_FETCH] set %s: %s, now %zu\n", e, cudaGetErrorString(le), v);
  }
  scan_ctx* s = new scan_ctx();
  s->c.device = cuda_device;
  s->c.stream = (cudaStream_t)cuda_stream;
  if (s->c.counters.ensure(sizeof(Counters)) != cudaSuccess) { delete s; return SCAN_E_OOM; }
  *out = s;
  return SCAN_OK;
}

static void release_all(Ctx& c) {
  DevBuf* bufs[] = {&c.own_dur, &c.own_kind, &c.own_meta, &c.own_comm, &c.own_pay, &c.rank_off, &c.coff, &c.cmem, &c.ccls,
                    &c.rcomm_off, &c.rcomm, &c.nbc_off, &c.nbc, &c.tile_rank, &c.tile_start, &c.rank_tile0, &c.tile_order, &c.t_nkeys,
                    &c.t_keys, &c.t_cnt, &c.t_pref, &c.t_ncomm, &c.t_niter, &c.t_last, &c.t_commpre, &c.t_iterpre,
                    &c.t_prevj, &c.r_nkeys, &c.r_keys, &c.r_cnt, &c.r_ncomm, &c.r_niter, &c.r_ncomp, &c.r_lastit,
                    &c.r_comm_off, &c.r_comp_off, &c.r_bits_off, &c.bitmap, &c.bitpre, &c.bmsum, &c.counters, &c.ch_nmax,
                    &c.ch_nmin, &c.ch_base, &c.ch_slot, &c.ch_nsend, &c.ch_nrecv, &c.inst_c, &c.wait_c, &c.cdur, &c.cop,
                    &c.slots, &c.lk_key, &c.inst_rec, &c.citer, &c.nbp, &c.nbp_n,
                    &c.rk_sum, &c.bits, &c.cref, &c.cl_J, &c.cl_max, &c.cl_min, &c.wd_total, &c.wd_slow, &c.wd_cand,
                    &c.wd_frac, &c.wl_joined, &c.wl_late, &c.wl_frac, &c.wl_verdict, &c.wl_link_slow, &c.ewc, &c.ewp,
                    &c.lk_n, &c.lk_used, &c.lk_medp, &c.lk_medt, &c.lk_bw, &c.lk_slow, &c.lk_dir, &c.lk_elig,
                    &c.lb_label, &c.lb_rkind, &c.lb_rrank, &c.lb_rsrc, &c.lb_depth, &c.lb_twait, &c.scratch,
                    &c.st_tile0, &c.st_npos, &c.role_comm, &c.role_slot, &c.role_type, &c.ncroles, &c.ft_cols,
                    &c.ft_base, &c.ft_last, &c.st_tot, &c.p2p_rbase, &c.dlate, &c.dinfo, &c.ft_posA, &c.ft_posB,
                    &c.ft_posK, &c.eidx, &c.tile_stage, &c.xbase, &c.g_base, &c.g_slot,
                    &c.g_nmax, &c.g_nmin, &c.g_k0, &c.p2p_eslot, &c.xe_off, &c.xe_col, &c.xbig, &c.own_start, &c.al_tend, &c.al_aend, &c.al_anct,
                    &c.al_anco, &c.al_level, &c.al_nanc, &c.al_resid, &c.al_flag, &c.al_start, &c.al_ranks, &c.al_tgt, &c.x_send, &c.x_recv, &c.x_recv2, &c.x_ep, &c.x_stage, &c.headtail, &c.lk_sendmap, &c.lk_recvmap, &c.al_xs, &c.al_xr, &c.al_row, &c.al_lt, &c.al_init, &c.al_bx, &c.al_bnd, &c.bl_xs, &c.bl_xr, &c.bl_gbase, &c.bl_ext, &c.al_imax, &c.al_vbits, &c.al_seg, &c.bl_seg, &c.bl_inst, &c.bl_pa, &c.bl_pb, &c.bl_root, &c.bl_last, &c.bl_rank, &c.bl_rk};
  for (DevBuf* b : bufs) b->release();
}

void scan_destroy(scan_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->c.device);
  if (ctx->c.stream) cudaStreamSynchronize(ctx->c.stream);
  for (auto& p : ctx->c.pend) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
  for (auto e : ctx->c.evpool) cudaEventDestroy(e);
  shard_release(ctx->c);
  stream_release(ctx->c);
  json_release(ctx->c);
  release_all(ctx->c);
  delete ctx;
}

const char* scan_last_error(const scan_ctx* ctx) { return ctx ? ctx->c.err.c_str() : "null context"; }

uint64_t scan_kernel_launches(const scan_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

scan_status scan_set_timing(scan_ctx* ctx, int enable) {
  if (!ctx) return SCAN_E_INVALID_ARG;
  ctx->c.timing = enable != 0;
  return SCAN_OK;
}

void scan_timing_reset(scan_ctx* ctx) {
  if (!ctx) return;
  Ctx& c = ctx->c;
  cudaStreamSynchronize(c.stream);
  resolve_timing(c);
  for (auto& x : c.kms) x = 0;
  for (auto& x : c.kcnt) x = 0;
}

int scan_kernel_timing(scan_ctx* ctx, int i, const char** name, double* total_ms, uint64_t* launches) {
  if (!ctx) return 0;
  Ctx& c = ctx->c;
  if (!c.pend.empty()) { cudaStreamSynchronize(c.stream); resolve_timing(c); }
  if (i >= 0 && i < (int)c.knames.size()) {
    if (name) *name = c.knames[i].c_str();
    if (total_ms) *total_ms = c.kms[i];
    if (launches) *launches = c.kcnt[i];
  }
  return (int)c.knames.size();
}

// ----------------------------------------------------------------------------- A0 ingest
scan_status scan_load_events(scan_ctx* ctx, const scan_topology* topo, const scan_comm_table* comms,
                             const scan_event_columns* cols, uint32_t flags) {
  if (!ctx || !topo || !comms || !cols) return SCAN_E_INVALID_ARG;
  Ctx& c = ctx->c;
  CK(cudaSetDevice(c.device));
  c.loaded = c.matched = c.detected = c.localized = false;
  c.fused_used = false; c.tiles_ready = false; c.xwait_pending = false; c.aligned = false;
  ++c.gen; ++c.load_id; c.blamed = false;
  if (c.stream_mode) { stream_release(c); c.stream_mode = false; }
  c.d_start = nullptr;
  c.err.clear();
  if (topo->tp < 1 || topo->pp < 1 || topo->dp < 1 || topo->rank_order != 0) {
    c.err = "topology: tp, pp, dp must be >= 1 and rank_order 0";
    return SCAN_E_INVALID_ARG;
  }
  const uint64_t W64 = (uint64_t)topo->tp * topo->pp * topo->dp;
  if (W64 > 65535) { c.err = "world size > 65535 unsupported"; return SCAN_E_UNSUPPORTED; }
  if (topo->dp > 32) { c.err = "dp > 32 unsupported by the stage-1 register network"; return SCAN_E_UNSUPPORTED; }
  const int W = (int)W64;
  if ((uint64_t)comms->n_comms + W64 * W64 >= (1ull << 32)) { c.err = "n_comms + world^2 must be < 2^32"; return SCAN_E_UNSUPPORTED; }
  if (!cols->rank_offsets || (cols->n_events && (!cols->dur_ns || !cols->kind_op || !cols->meta || !cols->comm || !cols->payload_bytes))) {
    c.err = "missing event column"; return SCAN_E_INVALID_ARG;
  }
  if (comms->n_comms && (!comms->offsets || !comms->members)) { c.err = "missing comm table"; return SCAN_E_INVALID_ARG; }
  const uint64_t N = cols->n_events;
  std::vector<uint64_t> ro(cols->rank_offsets, cols->rank_offsets + W + 1);
  if (ro[0] != 0 || ro[W] != N) { c.err = "rank_offsets must start at 0 and end at n_events"; return SCAN_E_INVALID_ARG; }
  for (int r = 0; r < W; ++r) {
    if (ro[r + 1] < ro[r]) { c.err = "rank_offsets not monotone"; return SCAN_E_INVALID_ARG; }
    if (ro[r + 1] - ro[r] >= (1ull << 31)) { c.err = "a rank holds >= 2^31 events"; return SCAN_E_UNSUPPORTED; }
  }
  // comm table checks + stage-2 class per communicator (reading R12), rank -> comms CSR,
  // collective neighbour lists (for the wait-for edge arrays)
  const uint32_t nc = comms->n_comms;
  // n_comms == 0 accepts offsets == NULL (nothing to read)
  std::vector<uint64_t> coff = nc ? std::vector<uint64_t>(comms->offsets, comms->offsets + nc + 1) : std::vector<uint64_t>{0};
  if (coff[0] != 0) { c.err = "comm offsets must start at 0"; return SCAN_E_INVALID_ARG; }
  std::vector<uint32_t> cmem(comms->members, comms->members + coff[nc]);
  std::vector<uint8_t> ccls(nc, 0);
  std::vector<std::vector<uint32_t>> rcl(W);
  const int TP = topo->tp, DP = topo->dp;
  for (uint32_t k = 0; k < nc; ++k) {
    if (coff[k + 1] < coff[k]) { c.err = "comm offsets not monotone"; return SCAN_E_INVALID_ARG; }
    const uint64_t b = coff[k], e = coff[k + 1];
    for (uint64_t q = b; q < e; ++q) {
      if (cmem[q] >= (uint32_t)W || (q > b && cmem[q] <= cmem[q - 1])) {
        c.err = "comm members must be ascending ranks < world"; return SCAN_E_INVALID_ARG;
      }
      rcl[cmem[q]].push_back(k);
    }
    const uint64_t n = e - b;
    if (n == 0) continue;
    const uint32_t r0 = cmem[b];
    if (TP >= 2 && n == (uint64_t)TP && r0 % TP == 0) {
      bool ok = true;
      for (int t = 0; t < TP; ++t) ok &= cmem[b + t] == r0 + (uint32_t)t;
      if (ok) { ccls[k] = 1; continue; }
    }
    if (DP >= 2 && n == (uint64_t)DP && (r0 / TP) % DP == 0) {
      bool ok = true;
      for (int d = 0; d < DP; ++d) ok &= cmem[b + d] == r0 + (uint32_t)(TP * d);
      if (ok) ccls[k] = 2;
    }
  }
  std::vector<uint32_t> rco(W + 1, 0), rcm;
  std::vector<uint64_t> nbo(W + 1, 0);
  std::vector<uint32_t> nb;
  for (int r = 0; r < W; ++r) {
    rco[r] = (uint32_t)rcm.size();
    rcm.insert(rcm.end(), rcl[r].begin(), rcl[r].end());
    std::vector<uint32_t> u;
    for (uint32_t k : rcl[r]) u.insert(u.end(), cmem.begin() + coff[k], cmem.begin() + coff[k + 1]);
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    nbo[r] = nb.size();
    for (uint32_t x : u) if (x != (uint32_t)r) nb.push_back(x);
  }
  rco[W] = (uint32_t)rcm.size();
  nbo[W] = nb.size();
  // tiles: TILE_EV consecutive events of one rank
  std::vector<uint32_t> trank, rt0(W + 1, 0);
  std::vector<uint64_t> tstart;
  for (int r = 0; r < W; ++r) {
    rt0[r] = (uint32_t)trank.size();
    for (uint64_t s = ro[r]; s < ro[r + 1]; s += TILE_EV) { trank.push_back((uint32_t)r); tstart.push_back(s); }
  }
  rt0[W] = (uint32_t)trank.size();
  // interleaved processing order of the tiles: chunk 0 of every rank, then chunk 1, ... -- the members
  // of an instance are then processed at about the same time, so the general path's per-instance
  // gathers (records) and scatters (member slots) meet in L2 instead of each fetching the sector
  std::vector<uint32_t> torder;
  torder.reserve(trank.size());
  {
    uint32_t maxc = 0;
    for (uint64_t r = 0; r < W; ++r) maxc = std::max(maxc, rt0[r + 1] - rt0[r]);
    for (uint32_t k = 0; k < maxc; ++k)
      for (uint64_t r = 0; r < W; ++r)
        if (rt0[r] + k < rt0[r + 1]) torder.push_back(rt0[r] + k);
  }
  c.TP = topo->tp; c.PP = topo->pp; c.DP = topo->dp; c.W = W; c.n_comms = nc; c.N = N; c.flags = flags;
  c.h_ccls = ccls; c.h_coff = coff; c.h_cmem = cmem; c.h_rcomm = rcm; c.h_rcomm_off = rco;
  {  // cross collectives (not TP/DP class) with <= 128 members: edge column of member q waiting on
     // member t (the search k_cross_reduce would do per wait-for edge; all co-members are neighbours)
    std::vector<uint64_t> xoff(std::max<uint32_t>(nc, 1), ~0ull);
    std::vector<uint32_t> xcol;
    for (uint32_t k = 0; k < nc; ++k) {
      const uint64_t b = coff[k], n = coff[k + 1] - b;
      if (ccls[k] == 1 || ccls[k] == 2 || n < 2 || n > 128) continue;
      xoff[k] = xcol.size();
      for (uint64_t q = 0; q < n; ++q) {
        const uint32_t r = cmem[b + q];
        for (uint64_t t = 0; t < n; ++t) {
          const uint32_t L = cmem[b + t];
          auto b0 = nb.begin() + nbo[r], b1 = nb.begin() + nbo[r + 1];
          auto it = std::lower_bound(b0, b1, L);
          xcol.push_back(q == t || it == b1 || *it != L ? 0u : (uint32_t)(it - nb.begin()));
        }
      }
    }
    if (xcol.empty()) xcol.push_back(0);
    std::vector<uint32_t> big;
    for (uint32_t k = 0; k < nc; ++k)
      if (ccls[k] != 1 && ccls[k] != 2 && coff[k + 1] - coff[k] > 32) big.push_back(k);
    c.n_big = (uint32_t)big.size();
    if (big.empty()) big.push_back(0);
    scan_status st0;
    if ((st0 = upload(c, c.xe_off, xoff)) || (st0 = upload(c, c.xe_col, xcol)) || (st0 = upload(c, c.xbig, big))) return st0;
  }
  c.h_rank_off = ro; c.h_rank_tile0 = rt0; c.n_tiles = trank.size(); c.nnz_c = nb.size();
  scan_status st;
  if ((st = upload(c, c.rank_off, ro)) || (st = upload(c, c.coff, coff)) || (st = upload(c, c.cmem, cmem)) ||
      (st = upload(c, c.ccls, ccls)) || (st = upload(c, c.rcomm_off, rco)) || (st = upload(c, c.rcomm, rcm)) ||
      (st = upload(c, c.nbc_off, nbo)) || (st = upload(c, c.nbc, nb)) || (st = upload(c, c.tile_rank, trank)) ||
      (st = upload(c, c.tile_start, tstart)) || (st = upload(c, c.rank_tile0, rt0)) || (st = upload(c, c.tile_order, torder)))
    return st;
  // fused-path (K9) tables: every stage block SPMD-compatible? role -> communicator / slot
  {
    c.spmd = false;
    const uint32_t R = (uint32_t)(topo->tp * topo->dp);
    bool ok = N > 0 && R <= 256;
    std::vector<uint32_t> rcmm((size_t)W * CROLES, NONE32), rslt((size_t)W * CROLES, NONE32), ncr(topo->pp, 0);
    std::vector<uint8_t> rty((size_t)topo->pp * ROLES, 0);
    std::vector<uint32_t> stt0(topo->pp + 1, 0), stnp(topo->pp, 0);
    bool aligned = true, aligned8 = true;
    for (int r = 0; r < W; ++r) { aligned &= (ro[r] % 4) == 0; aligned8 &= (ro[r] % 8) == 0; }
    for (int s = 0; ok && s < topo->pp; ++s) {
      const uint32_t r0 = s * R;
      const uint64_t ns = ro[r0 + 1] - ro[r0];
      if (rcl[r0].size() > (size_t)CROLES) { ok = false; break; }
      ncr[s] = (uint32_t)rcl[r0].size();
      for (uint32_t q = 0; q < ncr[s]; ++q) {
        const uint8_t k = ccls[rcl[r0][q]];
        rty[s * ROLES + q] = k == 1 ? 1 : (k == 2 ? 2 : 3);
      }
      for (uint32_t r = r0; ok && r < r0 + R; ++r) {
        if (ro[r + 1] - ro[r] != ns || rcl[r].size() != ncr[s]) { ok = false; break; }
        for (uint32_t q = 0; q < ncr[s]; ++q) {
          const uint32_t k = rcl[r][q];
          if (ccls[k] != ccls[rcl[r0][q]]) { ok = false; break; }
          rcmm[(size_t)r * CROLES + q] = k;
          rslt[(size_t)r * CROLES + q] = (uint32_t)(std::lower_bound(cmem.begin() + coff[k], cmem.begin() + coff[k + 1], r) -
                                                    (cmem.begin() + coff[k]));
        }
      }
      stnp[s] = (uint32_t)ns;
    }
    uint32_t ncrm = 1;
    for (int s = 0; s < topo->pp; ++s) ncrm = std::max(ncrm, ncr[s]);
    // edge slot of every TP-group / DP-group partner in the rank's collective neighbour list
    std::vector<uint32_t> eidx;
    if (ok) {
      const int TPn = topo->tp, DPn = topo->dp, E = TPn + DPn;
      eidx.assign((size_t)W * E, 0);
      for (int r = 0; r < W && ok; ++r) {
        const int t = r % TPn, d = (r / TPn) % DPn, s = r / (TPn * DPn);
        for (int q = 0; q < E; ++q) {
          const int partner = q < TPn ? (q + TPn * (d + DPn * s)) : (t + TPn * ((q - TPn) + DPn * s));
          if (partner == r) continue;
          auto b0 = nb.begin() + nbo[r], b1 = nb.begin() + nbo[r + 1];
          auto it = std::lower_bound(b0, b1, (uint32_t)partner);
          eidx[(size_t)r * E + q] = (it != b1 && *it == (uint32_t)partner) ? (uint32_t)(it - nb.begin()) : 0u;
        }
      }
    }
    if (ok) {
      const bool tp_pow2 = topo->tp <= 32 && (32 % topo->tp) == 0;
      c.fused_t = tp_pow2 && R <= 256 && c.fused_variant != 0;
      uint32_t T = ((c.fused_t ? fused_t_tile_events() : 16384u) / R) / 32u * 32u;
      if (const char* e = std::getenv("MS_FT_T")) T = (uint32_t)std::atoi(e) / 32u * 32u;  // experiment: tile positions
      T = std::max(64u, std::min(1024u, T));
      if (T < 128) T = 64;  // below 128 positions the load lane mapping needs a power of two
      // two CTAs per SM: keep the fused kernel's shared memory under ~110 KB
      auto smem = [&](uint32_t t) {
        return c.fused_t ? fused_t_smem_bytes(t, R, topo->tp, topo->dp, ncrm) : fused_smem_bytes(t, R, topo->tp, topo->dp, ncrm);
      };
      const size_t cap = c.fused_t ? fused_t_smem_cap() : 110u * 1024u;  // 2 (generic) / FT_MINB (transposed) CTAs per SM
      while (T > 32 && smem(T) > cap) T = T > 128 ? T - 32 : T / 2;  // below 128: powers of two (load lane mapping)
      if (std::getenv("MS_FT_T")) std::fprintf(stderr, "[MS_FT_T] tile positions %u, shared memory %zu of %zu\n", T, smem(T), cap);
      // the persistent TMA-fed kernel (k_stage.cu): 16-byte-aligned rank rows, R <= 128; its own tile size
      c.use_stage = false;
      const char* sge = std::getenv("MS_STAGE");  // experimental until it beats k_fused_t: variant 2 or MS_STAGE=1
      if (aligned && c.fused_t && (c.fused_variant == 2 || (c.fused_variant == -1 && sge && std::atoi(sge) == 1))) {
        const uint32_t Ts = stage_tile(R, (uint32_t)topo->tp, (uint32_t)topo->dp, ncrm, (uint32_t)topo->pp);
        if (Ts) { c.use_stage = true; T = Ts; }
      }
      c.NCRM = ncrm;
      if ((st = upload(c, c.eidx, eidx))) return st;
      uint32_t nt = 0;
      for (int s = 0; s < topo->pp; ++s) { stt0[s] = nt; nt += (stnp[s] + T - 1) / T; }
      stt0[topo->pp] = nt;
      c.FT = T; c.FR = R; c.n_ftiles = nt; c.h_st_tile0 = stt0; c.h_st_npos = stnp; c.rows_aligned = aligned; c.rows_aligned8 = aligned8;
      std::vector<uint8_t> tstage(nt);
      for (int s = 0; s < topo->pp; ++s) for (uint32_t t = stt0[s]; t < stt0[s + 1]; ++t) tstage[t] = (uint8_t)s;
      if (topo->pp > 255) ok = false;
      if ((st = upload(c, c.tile_stage, tstage))) return st;
      if ((st = upload(c, c.st_tile0, stt0)) || (st = upload(c, c.st_npos, stnp)) || (st = upload(c, c.role_comm, rcmm)) ||
          (st = upload(c, c.role_slot, rslt)) || (st = upload(c, c.role_type, rty)) || (st = upload(c, c.ncroles, ncr)))
        return st;
      c.spmd = ok && nt > 0;
    }
  }
  // event columns
  if (flags & SCAN_DEVICE_PTRS) {
    const void* ptrs[] = {cols->dur_ns, cols->kind_op, cols->meta, cols->comm, cols->payload_bytes};
    for (const void* p : ptrs)
      if (N && ((uintptr_t)p & 15)) { c.err = "device columns must be 16-byte aligned"; return SCAN_E_INVALID_ARG; }
    c.d_dur = cols->dur_ns; c.d_kind = cols->kind_op; c.d_meta = cols->meta; c.d_comm = cols->comm; c.d_pay = cols->payload_bytes;
    if (cols->start_ns && ((uintptr_t)cols->start_ns & 15)) { c.err = "device columns must be 16-byte aligned"; return SCAN_E_INVALID_ARG; }
    c.d_start = cols->start_ns;
  } else {
    CK(c.own_dur.ensure(N * 4)); CK(c.own_kind.ensure(N * 2)); CK(c.own_meta.ensure(N * 2));
    CK(c.own_comm.ensure(N * 4)); CK(c.own_pay.ensure(N * 4));
    if (N) {
      CK(cudaMemcpyAsync(c.own_dur.p, cols->dur_ns, N * 4, cudaMemcpyHostToDevice, c.stream));
      CK(cudaMemcpyAsync(c.own_kind.p, cols->kind_op, N * 2, cudaMemcpyHostToDevice, c.stream));
      CK(cudaMemcpyAsync(c.own_meta.p, cols->meta, N * 2, cudaMemcpyHostToDevice, c.stream));
      CK(cudaMemcpyAsync(c.own_comm.p, cols->comm, N * 4, cudaMemcpyHostToDevice, c.stream));
      CK(cudaMemcpyAsync(c.own_pay.p, cols->payload_bytes, N * 4, cudaMemcpyHostToDevice, c.stream));
    }
    if (cols->start_ns) {  // only the timeline alignment reads start times
      CK(c.own_start.ensure(N * 8));
      if (N) CK(cudaMemcpyAsync(c.own_start.p, cols->start_ns, N * 8, cudaMemcpyHostToDevice, c.stream));
      c.d_start = c.own_start.as<int64_t>();
    }
    c.d_dur = c.own_dur.as<uint32_t>(); c.d_kind = c.own_kind.as<uint16_t>(); c.d_meta = c.own_meta.as<uint16_t>();
    c.d_comm = c.own_comm.as<uint32_t>(); c.d_pay = c.own_pay.as<uint32_t>();
  }
  CK(cudaStreamSynchronize(c.stream));
  c.loaded = true;
  return SCAN_OK;
}

// ----------------------------------------------------------------------------- shared stages
}  // extern "C"

namespace {

const scan_detect_config kDefDetect{3, 2, 50000, 3, 10, 10, 0, 0, 0};
const scan_localize_config kDefLocalize{100000, 7, 10, 7, 10, 10, 3, 0, 0, 100000};

}  // namespace

// per-rank / channel workspaces and counter reset (both paths)
scan_status ms::prep_ws(Ctx& c, bool tiles) {
  const uint64_t T = std::max<uint64_t>(c.n_tiles, 1), W = c.W;
  if (tiles) {
    CK(c.t_nkeys.ensure(T * 4)); CK(c.t_keys.ensure(T * KCAP * 4)); CK(c.t_cnt.ensure(T * KCAP * 4));
    CK(c.t_pref.ensure(T * KCAP * 4)); CK(c.t_ncomm.ensure(T * 4)); CK(c.t_niter.ensure(T * 4)); CK(c.t_last.ensure(T * 4));
    CK(c.t_commpre.ensure(T * 4)); CK(c.t_iterpre.ensure(T * 4)); CK(c.t_prevj.ensure(T * 4));
  }
  CK(c.r_nkeys.ensure(W * 4)); CK(c.r_keys.ensure(W * RCAP * 4)); CK(c.r_cnt.ensure(W * RCAP * 4));
  CK(c.r_ncomm.ensure(W * 4)); CK(c.r_niter.ensure(W * 4)); CK(c.r_ncomp.ensure(W * 4));
  CK(c.r_comm_off.ensure((W + 1) * 8)); CK(c.r_comp_off.ensure((W + 1) * 8)); CK(c.r_bits_off.ensure((W + 1) * 8));
  c.n_bm_words = (W * W + 31) / 32;
  CK(c.bitmap.ensure(c.n_bm_words * 4)); CK(c.bitpre.ensure(c.n_bm_words * 4));
  const uint64_t ch_cap = c.n_comms + W * RCAP;
  CK(c.ch_nmax.ensure(ch_cap * 4)); CK(c.ch_nmin.ensure(ch_cap * 4));
  CK(c.nbp.ensure(W * PCAP * 4)); CK(c.nbp_n.ensure(W * 4));
  Counters z{};
  z.bad_event = ~0ull;
  z.min_niter = ~0u;
  CK(cudaMemcpyAsync(c.counters.p, &z, sizeof(Counters), cudaMemcpyHostToDevice, c.stream));
  queue_fill(c, c.ch_nmax.p, ch_cap * 4, 0);
  queue_fill(c, c.ch_nmin.p, ch_cap * 4, 0xFF);
  queue_fill(c, c.bitmap.p, c.n_bm_words * 4, 0);
  return SCAN_OK;
}

namespace {

// after the per-rank census (general: k_rank_scan, fused: k_fused_census) + k_rank_prefix:
// read totals, build channel bases, allocate the per-event / per-instance buffers.
scan_status channels_and_buffers(Ctx& c, bool fused) {
  scan_status st = sync_read(c);
  if (st) return st;
  if (fused && (c.hc.overflow & 32u)) return 2;  // not SPMD: caller falls back
  if (c.hc.bad_event != ~0ull) {
    std::ostringstream m;
    m << "schema error at event " << c.hc.bad_event << " (kind > 6, comm id out of range, rank not a member, or bad peer)";
    c.err = m.str();
    return SCAN_E_SCHEMA;
  }
  if (c.hc.overflow & 7u) {
    if (fused) return 2;
    c.err = "capacity exceeded: " + std::string((c.hc.overflow & 1) ? "more than 32 channels in a 2048-event tile " : "") +
            ((c.hc.overflow & 2) ? "more than 256 channels on a rank " : "") + ((c.hc.overflow & 4) ? "more than 32 P2P peers on a rank" : "");
    return SCAN_E_UNSUPPORTED;
  }
  const uint64_t W = c.W;
  c.n_p2p = c.hc.n_p2p; c.NCH = c.n_comms + c.n_p2p; c.n_comm = c.hc.n_comm; c.n_comp = c.hc.n_comp;
  c.NIT = c.hc.max_niter; c.n_iters = c.hc.n_iters; c.max_ncomp = c.hc.max_ncomp; c.n_bits_words = c.hc.n_bits_words;
  CK(c.ch_base.ensure((c.NCH + 1) * 8)); CK(c.ch_slot.ensure((c.NCH + 1) * 8)); CK(c.xbase.ensure((c.NCH + 1) * 8));
  CK(c.ch_nsend.ensure(std::max<uint64_t>(2 * c.n_p2p, 1) * 4)); CK(c.ch_nrecv.ensure(std::max<uint64_t>(2 * c.n_p2p, 1) * 4));
  if (c.n_p2p) {
    CK(cudaMemsetAsync(c.ch_nsend.p, 0, 2 * c.n_p2p * 4, c.stream));
    CK(cudaMemsetAsync(c.ch_nrecv.p, 0, 2 * c.n_p2p * 4, c.stream));
  }
  c.launches += timed(c, "k_channels", [&] { return launch_p2p_channels(c); });
  if ((st = sync_read(c))) return st;
  if (c.hc.n_instances >= 0xFFFFFFFFull) { c.err = "more than 2^32-1 instances"; return SCAN_E_UNSUPPORTED; }
  c.n_inst = c.hc.n_instances; c.n_slots = c.hc.n_slots; c.p2p_slot0 = c.hc.p2p_slot0; c.p2p_inst0 = c.hc.p2p_inst0;
  c.n_xinst = c.hc.n_xinst;
  return alloc_match_buffers(c, fused);
}

}  // namespace

// per-event / per-slot / per-instance buffers once the channel tables are final
scan_status ms::alloc_match_buffers(Ctx& c, bool fused) {
  const uint64_t W = c.W;
  CK(c.inst_c.ensure(c.n_comm * 4)); CK(c.wait_c.ensure(c.n_comm * 4));
  if (!fused) { CK(c.cdur.ensure(c.n_comp * 4)); CK(c.cop.ensure(c.n_comp * 2)); }
  if ((uint64_t)c.it_off + c.n_iters >= SLOT_MAX_ITERS) { c.err = "more than 2^28 iterations"; return SCAN_E_UNSUPPORTED; }
  CK(c.slots.ensure(c.n_slots * 16));
  CK(c.lk_key.ensure(std::max<uint64_t>(c.n_inst - c.p2p_inst0, 1) * 8));
  if (fused) CK(c.p2p_rbase.ensure(W * 16 * 4));
  CK(c.inst_rec.ensure(c.n_inst * 16));
  const uint32_t NIT1 = c.NIT + 1;
  CK(c.citer.ensure(W * NIT1 * 4));
  const uint64_t n = W * NIT1;
  if (fused) return SCAN_OK;  // citer (compute index of each iteration start) is read by the general path only
  flush_fills(c);
  k_citer_fill<<<(unsigned)((n + 255) / 256), 256, 0, c.stream>>>(c.W, NIT1, c.r_ncomp.as<uint32_t>(), c.citer.as<uint32_t>());
  c.launches += 1;
  return SCAN_OK;
}

scan_status ms::alloc_detect(Ctx& c) {
  const scan_detect_config& d = c.dcfg;
  c.NW = d.window_iters ? std::max<uint32_t>(1, (c.n_iters + d.window_iters - 1) / d.window_iters) : 1;
  const uint64_t ncl = (uint64_t)c.TP * c.PP, items = (uint64_t)c.NW * c.W;
  CK(c.bits.ensure(std::max<uint64_t>(c.n_bits_words, 1) * 4));
  queue_fill(c, c.bits.p, std::max<uint64_t>(c.n_bits_words, 1) * 4, 0);
  if (d.want_ref) { CK(c.cref.ensure(std::max<uint64_t>(c.n_comp, 1) * 4)); queue_fill(c, c.cref.p, c.n_comp * 4, 0xFF); }
  CK(c.cl_J.ensure(ncl * 4)); CK(c.cl_max.ensure(ncl * 4)); CK(c.cl_min.ensure(ncl * 4));
  CK(c.wd_total.ensure(items * 4)); CK(c.wd_slow.ensure(items * 4)); CK(c.wd_cand.ensure(items)); CK(c.wd_frac.ensure(items * 8));
  return SCAN_OK;
}

scan_status ms::alloc_localize(Ctx& c) {
  const uint64_t items = (uint64_t)c.NW * c.W, nlk = (uint64_t)c.NW * c.n_p2p;
  const uint64_t nnz_tot = c.nnz_c + (uint64_t)c.W * PCAP;
  CK(c.wl_joined.ensure(items * 4)); CK(c.wl_late.ensure(items * 4)); CK(c.wl_frac.ensure(items * 8));
  CK(c.wl_verdict.ensure(items)); CK(c.wl_link_slow.ensure(items));
  CK(c.ewc.ensure(c.NW * nnz_tot * 8)); CK(c.rk_sum.ensure(3ull * c.W * 8));
  CK(c.lk_n.ensure(nlk * 4 + 4)); CK(c.lk_used.ensure(nlk + 1)); CK(c.lk_medp.ensure(nlk * 4 + 4));
  CK(c.lk_medt.ensure(nlk * 4 + 4)); CK(c.lk_bw.ensure(nlk * 8 + 8)); CK(c.lk_slow.ensure(nlk + 1));
  CK(c.lk_dir.ensure(nlk + 1)); CK(c.lk_elig.ensure(nlk + 1));
  CK(c.lb_label.ensure(items)); CK(c.lb_rkind.ensure(items)); CK(c.lb_rrank.ensure(items * 4));
  CK(c.lb_rsrc.ensure(items * 4)); CK(c.lb_depth.ensure(items * 4)); CK(c.lb_twait.ensure(items * 8));
  CK(c.scratch.ensure(std::max<size_t>(c.scratch.cap, (2 * items + c.NW + 2) * 4)));
  queue_fill(c, c.wl_joined.p, items * 4, 0);
  queue_fill(c, c.wl_late.p, items * 4, 0);
  queue_fill(c, c.wl_link_slow.p, items, 0);
  queue_fill(c, c.ewc.p, c.NW * nnz_tot * 8, 0);
  queue_fill(c, c.rk_sum.p, 3ull * c.W * 8, 0);
  queue_fill(c, c.lk_slow.p, nlk + 1, 0);
  queue_fill(c, c.scratch.as<uint32_t>() + 2 * items, (c.NW + 2) * 4, 0);
  return SCAN_OK;
}

namespace {

void fill_match(Ctx& c, scan_match_result* out) {
  if (!out) return;
  const bool sh = c.n_shards > 1;  // sharded: job-wide totals
  out->n_events = sh ? c.g_N : c.N; out->n_comm_events = sh ? c.g_ncomm : c.n_comm;
  out->n_compute_events = sh ? c.g_ncomp : c.n_comp;
  out->n_channels = c.NCH; out->n_p2p_channels = c.n_p2p; out->n_instances = c.n_inst;
  out->n_incomplete = c.hc.n_incomplete; out->n_kind_mismatch = c.hc.n_kind_mismatch;
  out->n_payload_mismatch = c.hc.n_payload_mismatch; out->n_iters = c.n_iters;
}

scan_status match_status(Ctx& c) {
  const bool reports = c.hc.n_incomplete || c.hc.n_kind_mismatch || c.hc.n_payload_mismatch;
  if (reports && (c.flags & SCAN_STRICT)) { c.err = "integrity: unmatched or inconsistent instances"; return SCAN_E_INTEGRITY; }
  return reports ? SCAN_PARTIAL : SCAN_OK;
}

scan_status detect_tail(Ctx& c, scan_detect_result* out) {
  const uint64_t ncl = (uint64_t)c.TP * c.PP;
  std::vector<uint32_t> J(ncl), mx(ncl);
  CK(cudaMemcpy(J.data(), c.cl_J.p, ncl * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(mx.data(), c.cl_max.p, ncl * 4, cudaMemcpyDeviceToHost));
  uint64_t mism = 0;
  if (c.DP >= 2) for (uint64_t i = 0; i < ncl; ++i) mism += J[i] != mx[i];
  if (out) {
    out->n_windows = c.NW; out->n_compared = c.hc.n_compared; out->n_slow = c.hc.n_slow;
    out->n_candidates = c.hc.n_candidates; out->n_class_mismatch = mism;
  }
  return SCAN_OK;
}

void fill_localize(Ctx& c, scan_localize_result* out) {
  if (!out) return;
  out->n_windows = c.NW; out->n_links = (uint64_t)c.NW * c.n_p2p; out->n_link_slow = c.hc.n_link_slow;
  out->n_compute_slow = c.hc.v_count[SCAN_V_COMPUTE_SLOW]; out->n_link_slow_ranks = c.hc.v_count[SCAN_V_LINK_SLOW];
  out->n_both = c.hc.v_count[SCAN_V_BOTH]; out->n_exonerated = c.hc.v_count[SCAN_V_EXONERATED];
  out->n_insufficient = c.hc.v_count[SCAN_V_INSUFFICIENT]; out->n_roots = c.hc.n_roots;
  out->n_victims = c.hc.n_victims; out->n_unattributed = c.hc.n_unattributed; out->n_edges = 0;
}

// ---- the general path, stage by stage
scan_status general_match(Ctx& c) {
  c.matched = c.detected = c.localized = false;
  scan_status st = prep_ws(c, true);
  if (st) return st;
  c.launches += timed(c, "k_tile_scan", [&] { return launch_tile_scan(c); });
  c.launches += timed(c, "k_rank_scan", [&] { return launch_rank_scan(c); });
  c.launches += timed(c, "k_rank_prefix", [&] { return launch_rank_prefix(c); });
  c.tiles_ready = true;
  c.fused_used = false;
  c.xwait_pending = false;
  if ((st = channels_and_buffers(c, false))) return st;
  c.launches += timed(c, "k_assign", [&] { return launch_assign(c); });
  c.launches += timed(c, "k_inst_reduce", [&] { return launch_inst_reduce(c); });
  if ((st = sync_read(c))) return st;
  c.matched = true;
  return SCAN_OK;
}

scan_status general_detect(Ctx& c) {
  c.detected = c.localized = false;
  scan_status st = alloc_detect(c);
  if (st) return st;
  Counters z = c.hc;
  z.n_compared = z.n_slow = z.n_candidates = z.n_class_mismatch = 0;
  CK(cudaMemcpyAsync(c.counters.p, &z, sizeof(Counters), cudaMemcpyHostToDevice, c.stream));
  const int l1 = timed(c, "k_stage1", [&] { return launch_stage1(c); });
  if (l1 < 0) { c.err = "stage 1: dp unsupported"; return SCAN_E_UNSUPPORTED; }
  c.launches += l1;
  c.launches += timed(c, "k_stage1_counts", [&] { return launch_stage1_counts(c); });
  if ((st = sync_read(c))) return st;
  c.detected = true;
  return SCAN_OK;
}

scan_status general_localize(Ctx& c) {
  c.localized = false;
  scan_status st = alloc_localize(c);
  if (st) return st;
  Counters z = c.hc;
  z.n_link_slow = z.n_roots = z.n_victims = z.n_unattributed = 0;
  for (auto& v : z.v_count) v = 0;
  CK(cudaMemcpyAsync(c.counters.p, &z, sizeof(Counters), cudaMemcpyHostToDevice, c.stream));
  c.launches += timed(c, "k_event_pass", [&] { return launch_event_pass(c); });
  c.launches += timed(c, "k_link_median", [&] { return launch_link_median(c); });
  c.launches += timed(c, "k_link_flags", [&] { return launch_link_flags(c); });
  c.launches += timed(c, "k_walk", [&] { return launch_verdict_walk(c); });
  if ((st = sync_read(c))) return st;
  if (c.hc.overflow & 24u) {
    c.err = "capacity exceeded: more than 16384 samples on a link / links in a direction class";
    return SCAN_E_UNSUPPORTED;
  }
  c.localized = true;
  return SCAN_OK;
}

}  // namespace

// ---- streaming fast path: the previous fused analysis of this context was on a trace with the same
// per-rank event counts (a new iteration of an SPMD job): the template, tile bases, channel tables
// and buffer sizes are reused; the fused kernel re-verifies every event against the cached
// template (a deviation is reported, never silently analysed). Partials only (partial_tail).
bool ms::sync_check_on() {
  static const bool on = [] { const char* e = std::getenv("MS_SYNC_CHECK"); return e && *e == '1'; }();
  return on;
}

void ms::sync_check(Ctx& c, const char* name) {
  const cudaError_t e = cudaStreamSynchronize(c.stream);
  if (e != cudaSuccess) std::fprintf(stderr, "[MS_SYNC_CHECK] %s: %s\n", name, cudaGetErrorString(e));
}

scan_status ms::fused_rerun(Ctx& c) {
  c.matched = c.detected = c.localized = false;
  scan_status st;
  if ((st = alloc_match_buffers(c, true)) || (st = alloc_detect(c)) || (st = alloc_localize(c))) return st;
  queue_fill(c, c.dlate.p, (uint64_t)c.n_ftiles * ((c.FR + 31) / 32) * 4 + 4, 0);
  queue_fill(c, c.wd_total.p, (uint64_t)c.NW * c.W * 4, 0);
  queue_fill(c, c.wd_slow.p, (uint64_t)c.NW * c.W * 4, 0);
  Counters z = c.hc;
  z.overflow = 0; z.bad_event = ~0ull;
  z.n_incomplete = z.n_kind_mismatch = z.n_payload_mismatch = 0;
  z.n_compared = z.n_slow = z.n_candidates = z.n_class_mismatch = 0;
  z.n_link_slow = z.n_roots = z.n_victims = z.n_unattributed = 0;
  for (auto& v : z.v_count) v = 0;
  CK(cudaMemcpyAsync(c.counters.p, &z, sizeof(Counters), cudaMemcpyHostToDevice, c.stream));
  c.launches += timed(c, "k_class_counts", [&] { return launch_class_counts(c); });
  c.launches += timed(c, stage_active(c) ? "k_stage" : "k_fused", [&] { return launch_fused(c); });
  c.launches += timed(c, "k_cross_reduce", [&] { return launch_cross_reduce(c); });
  c.launches += timed(c, "k_deferred", [&] { return launch_deferred(c); });
  if ((st = sync_read(c))) return st;
  if (c.hc.overflow & 32u) { c.err = "streaming: an iteration deviates from the cached SPMD template"; return SCAN_E_UNSUPPORTED; }
  c.matched = c.detected = c.localized = true;
  c.fused_used = true;
  return SCAN_OK;
}

// ---- the fused SPMD path (K9); returns 2 when the trace is not SPMD (caller falls back)
scan_status ms::fused_all(Ctx& c) {
  c.matched = c.detected = c.localized = false;
  c.xwait_pending = false;
  scan_status st = prep_ws(c, false);
  if (st) return st;
  CK(c.ft_cols.ensure((uint64_t)FCOLS * c.n_ftiles * 4)); CK(c.ft_base.ensure((uint64_t)FCOLS * c.n_ftiles * 4));
  CK(c.st_tot.ensure((uint64_t)c.PP * FCOLS * 4));
  CK(c.ft_posA.ensure((uint64_t)c.n_ftiles * c.FT * 4)); CK(c.ft_posB.ensure((uint64_t)c.n_ftiles * c.FT * 4));
  CK(c.ft_posK.ensure((uint64_t)c.n_ftiles * c.FT * 2));
  if (c.use_stage) CK(c.ft_tbase.ensure((uint64_t)c.n_ftiles * 40 * 4));
  c.launches += timed(c, "k_fused_prepass", [&] { return launch_fused_prepass(c); });
  c.launches += timed(c, "k_fused_census", [&] { return launch_fused_census(c); });
  c.launches += timed(c, "k_rank_prefix", [&] { return launch_rank_prefix(c); });
  c.tiles_ready = false;
  if ((st = channels_and_buffers(c, true))) return st;
  if ((st = alloc_detect(c)) || (st = alloc_localize(c))) return st;
  CK(c.dlate.ensure((uint64_t)c.n_ftiles * ((c.FR + 31) / 32) * 4 + 4));
  queue_fill(c, c.dlate.p, (uint64_t)c.n_ftiles * ((c.FR + 31) / 32) * 4 + 4, 0);
  CK(c.dinfo.ensure((uint64_t)c.n_ftiles * 16 + 16));
  Counters z = c.hc;
  z.n_compared = z.n_slow = z.n_candidates = z.n_class_mismatch = 0;
  z.n_link_slow = z.n_roots = z.n_victims = z.n_unattributed = 0;
  for (auto& v : z.v_count) v = 0;
  CK(cudaMemcpyAsync(c.counters.p, &z, sizeof(Counters), cudaMemcpyHostToDevice, c.stream));
  {
    const uint64_t items = (uint64_t)c.NW * c.W;
    queue_fill(c, c.wd_total.p, items * 4, 0);
    queue_fill(c, c.wd_slow.p, items * 4, 0);
  }
  c.launches += timed(c, "k_class_counts", [&] { return launch_class_counts(c); });
  c.launches += timed(c, "k_p2p_roles", [&] { return launch_p2p_roles(c); });
  c.launches += timed(c, stage_active(c) ? "k_stage" : "k_fused", [&] { return launch_fused(c); });
  c.launches += timed(c, "k_cross_reduce", [&] { return launch_cross_reduce(c); });
  c.launches += timed(c, "k_deferred", [&] { return launch_deferred(c); });
  if (c.partial_tail) {  // streaming: per-iteration partials only (stream.cu combines the window)
    if ((st = sync_read(c))) return st;
    if (c.hc.overflow & 32u) { c.err = "streaming needs an SPMD iteration (fused-pass verification failed)"; return SCAN_E_UNSUPPORTED; }
    c.matched = c.detected = c.localized = true;
    c.fused_used = true;
    return SCAN_OK;
  }
  c.launches += timed(c, "k_wd_finish", [&] { return launch_wd_finish(c); });
  // links and walk run before the SPMD verification result is read (one host sync less): on a
  // failed verification their inputs are garbage but in bounds, and the call reruns the general path
  c.launches += timed(c, "k_link_median", [&] { return launch_link_median(c); });
  c.launches += timed(c, "k_link_flags", [&] { return launch_link_flags(c); });
  c.launches += timed(c, "k_walk", [&] { return launch_verdict_walk(c); });
  if ((st = sync_read(c))) return st;
  if (c.hc.overflow & 32u) return 2;
  c.matched = c.detected = true;
  if (c.hc.overflow & 24u) {
    c.err = "capacity exceeded: more than 16384 samples on a link / links in a direction class";
    return SCAN_E_UNSUPPORTED;
  }
  c.localized = true;
  c.fused_used = true;
  c.xwait_pending = true;
  return SCAN_OK;
}

extern "C" {

// ----------------------------------------------------------------------------- A1-A3 match
scan_status scan_match_collectives(scan_ctx* ctx, scan_match_result* out) {
  if (!ctx) return SCAN_E_INVALID_ARG;
  Ctx& c = ctx->c;
  ++c.gen; c.blamed = false;
  if (!c.loaded) { c.err = "scan_match_collectives before scan_load_events"; return SCAN_E_ORDER; }
  if (c.n_shards > 1) { c.err = "a sharded context runs scan_analyze only"; return SCAN_E_UNSUPPORTED; }
  CK(cudaSetDevice(c.device));
  c.launches = 0;
  scan_status st = general_match(c);
  if (st) return st;
  fill_match(c, out);
  return match_status(c);
}

// ----------------------------------------------------------------------------- A4 detect
scan_status scan_detect(scan_ctx* ctx, const scan_detect_config* cfg, scan_detect_result* out) {
  if (!ctx) return SCAN_E_INVALID_ARG;
  Ctx& c = ctx->c;
  ++c.gen; c.blamed = false;
  if (!c.matched) { c.err = "scan_detect before scan_match_collectives"; return SCAN_E_ORDER; }
  CK(cudaSetDevice(c.device));
  scan_detect_config d = cfg ? *cfg : kDefDetect;
  if (d.slow_den == 0 || d.cand_den == 0) { c.err = "zero denominator"; return SCAN_E_INVALID_ARG; }
  if (c.fused_used) { c.err = "scan_detect after scan_analyze: call scan_match_collectives first"; return SCAN_E_ORDER; }
  c.dcfg = d;
  scan_status st = general_detect(c);
  if (st) return st;
  return detect_tail(c, out);
}

// ----------------------------------------------------------------------------- A5-A8 localize
scan_status scan_localize(scan_ctx* ctx, const scan_localize_config* cfg, scan_localize_result* out) {
  if (!ctx) return SCAN_E_INVALID_ARG;
  Ctx& c = ctx->c;
  ++c.gen; c.blamed = false;
  if (!c.detected || c.fused_used) { c.err = "scan_localize before scan_detect"; return SCAN_E_ORDER; }
  CK(cudaSetDevice(c.device));
  scan_localize_config L = cfg ? *cfg : kDefLocalize;
  if (L.late_den == 0 || L.bw_den == 0) { c.err = "zero denominator"; return SCAN_E_INVALID_ARG; }
  c.lcfg = L;
  scan_status st = general_localize(c);
  if (st) return st;
  fill_localize(c, out);
  return SCAN_OK;
}

// ----------------------------------------------------------------------------- A1-A8 fused
scan_status scan_analyze(scan_ctx* ctx, const scan_detect_config* dcfg, const scan_localize_config* lcfg,
                         scan_match_result* mres, scan_detect_result* dres, scan_localize_result* lres) {
  if (!ctx) return SCAN_E_INVALID_ARG;
  Ctx& c = ctx->c;
  ++c.gen; c.blamed = false;
  if (!c.loaded) { c.err = "scan_analyze before scan_load_events"; return SCAN_E_ORDER; }
  CK(cudaSetDevice(c.device));
  scan_detect_config d = dcfg ? *dcfg : kDefDetect;
  scan_localize_config L = lcfg ? *lcfg : kDefLocalize;
  if (d.slow_den == 0 || d.cand_den == 0 || L.late_den == 0 || L.bw_den == 0) { c.err = "zero denominator"; return SCAN_E_INVALID_ARG; }
  c.dcfg = d; c.lcfg = L;
  c.launches = 0;
  scan_status st = 2;
  if (c.n_shards > 1) {  // iteration-window shard of a multi-GPU job (shard.cu): collective call
    if ((st = sharded_all(c))) return st;
    fill_match(c, mres);
    if ((st = detect_tail(c, dres))) return st;
    fill_localize(c, lres);
    return match_status(c);
  }
  if (c.spmd && !c.force_general) {
    st = fused_all(c);
    if (st < 0) return st;
  }
  if (st == 2) {  // not SPMD (or forced): the general path
    c.launches = 0;
    if ((st = general_match(c)) || (st = general_detect(c)) || (st = general_localize(c))) return st;
  }
  fill_match(c, mres);
  if ((st = detect_tail(c, dres))) return st;
  fill_localize(c, lres);
  return match_status(c);
}

int scan_used_fused(const scan_ctx* ctx) { return ctx && ctx->c.fused_used ? 1 : 0; }

// ----------------------------------------------------------------------------- NEXT-1 alignment
scan_status scan_align(scan_ctx* ctx, const scan_align_config* cfg, scan_align_result* out) {
  if (!ctx) return SCAN_E_INVALID_ARG;
  Ctx& c = ctx->c;
  ++c.gen;
  if (!c.matched) { c.err = "scan_align before scan_analyze / scan_match_collectives"; return SCAN_E_ORDER; }
  // a sharded context aligns collectively (every shard calls): see align_all
  if (!c.d_start) { c.err = "scan_align needs start_ns at scan_load_events"; return SCAN_E_INVALID_ARG; }
  const int32_t ref = cfg ? cfg->reference : 0;
  if (ref < 0 || ref >= c.W) { c.err = "reference rank out of range"; return SCAN_E_INVALID_ARG; }
  CK(cudaSetDevice(c.device));
  scan_status st = ensure_tiles(c);
  if (st) return st;
  c.aligned = false;
  if ((st = align_all(c, ref, out))) return st;
  c.aligned = true;
  return SCAN_OK;
}

scan_status scan_fused_variant(scan_ctx* ctx, int variant) {
  if (!ctx || variant < -1 || variant > 2) return SCAN_E_INVALID_ARG;
  ctx->c.fused_variant = variant;
  return SCAN_OK;
}

scan_status scan_force_general(scan_ctx* ctx, int force) {
  if (!ctx) return SCAN_E_INVALID_ARG;
  ctx->c.force_general = force != 0;
  return SCAN_OK;
}

}  // extern "C"

// ----------------------------------------------------------------------------- exports
// general tile prefixes (per 2048-event tile: comm / iteration counts) for event-order work after a
// fused analysis: built once per analysis, outside the timed step
scan_status ms::ensure_tiles(Ctx& c) {
  if (c.tiles_ready) return SCAN_OK;
  const uint64_t T = std::max<uint64_t>(c.n_tiles, 1);
  CK(c.t_nkeys.ensure(T * 4)); CK(c.t_keys.ensure(T * KCAP * 4)); CK(c.t_cnt.ensure(T * KCAP * 4));
  CK(c.t_pref.ensure(T * KCAP * 4)); CK(c.t_ncomm.ensure(T * 4)); CK(c.t_niter.ensure(T * 4)); CK(c.t_last.ensure(T * 4));
  CK(c.t_commpre.ensure(T * 4)); CK(c.t_iterpre.ensure(T * 4)); CK(c.t_prevj.ensure(T * 4));
  launch_tile_scan(c);
  launch_rank_scan(c);
  CK(cudaStreamSynchronize(c.stream));
  CK(cudaGetLastError());
  c.tiles_ready = true;
  return SCAN_OK;
}

namespace {

struct OutDesc { const DevBuf* buf; uint64_t off_bytes; uint64_t bytes; int stage; };

// host-side assembly of small tables (channels, edges, per-link ids)
scan_status host_table(Ctx& c, scan_output which, std::vector<uint8_t>& out) {
  auto d2h = [&](const DevBuf& b, uint64_t off, uint64_t bytes, void* dst) -> cudaError_t {
    if (!bytes) return cudaSuccess;
    return cudaMemcpy(dst, (const uint8_t*)b.p + off, bytes, cudaMemcpyDeviceToHost);
  };
  const uint64_t NCH = c.NCH, np = c.n_p2p, nc = c.n_comms;
  const bool sh = c.n_shards > 1;
  std::vector<uint32_t> psrc(np), pdst(np);
  CK(d2h(c.ch_nsend, np * 4, np * 4, psrc.data()));
  CK(d2h(c.ch_nrecv, np * 4, np * 4, pdst.data()));
  auto put = [&](const auto& v) {
    out.resize(v.size() * sizeof(v[0]));
    if (!v.empty()) std::memcpy(out.data(), v.data(), out.size());
  };
  switch (which) {
    case SCAN_OUT_CH_KIND: { std::vector<uint8_t> v(NCH, 0); for (uint64_t i = nc; i < NCH; ++i) v[i] = 1; put(v); return SCAN_OK; }
    case SCAN_OUT_CH_A: { std::vector<uint32_t> v(NCH); for (uint64_t i = 0; i < NCH; ++i) v[i] = i < nc ? (uint32_t)i : psrc[i - nc]; put(v); return SCAN_OK; }
    case SCAN_OUT_CH_B: { std::vector<uint32_t> v(NCH); for (uint64_t i = 0; i < NCH; ++i) v[i] = i < nc ? NONE32 : pdst[i - nc]; put(v); return SCAN_OK; }
    case SCAN_OUT_CH_NMEM: {
      std::vector<uint64_t> co(nc + 1);
      CK(d2h(c.coff, 0, (nc + 1) * 8, co.data()));
      std::vector<uint32_t> v(NCH);
      for (uint64_t i = 0; i < NCH; ++i) v[i] = i < nc ? (uint32_t)(co[i + 1] - co[i]) : 2;
      put(v); return SCAN_OK;
    }
    // sharded contexts: the job-wide tables (the kernels' ch_* are this shard's shifted / local ones)
    case SCAN_OUT_CH_NMAX: { std::vector<uint32_t> v(NCH); CK(d2h(sh ? c.g_nmax : c.ch_nmax, 0, NCH * 4, v.data())); put(v); return SCAN_OK; }
    case SCAN_OUT_CH_NMIN: { std::vector<uint32_t> v(NCH); CK(d2h(sh ? c.g_nmin : c.ch_nmin, 0, NCH * 4, v.data())); put(v); return SCAN_OK; }
    case SCAN_OUT_CH_BASE: { std::vector<uint64_t> v(NCH); CK(d2h(sh ? c.g_base : c.ch_base, 0, NCH * 8, v.data())); put(v); return SCAN_OK; }
    case SCAN_OUT_CH_SHARD_K0: {
      std::vector<uint64_t> v(NCH, 0);
      if (sh) v = c.h_shard_k0;
      put(v); return SCAN_OK;
    }
    case SCAN_OUT_CH_SHARD_N: {
      std::vector<uint32_t> v(NCH);
      if (sh) v = c.h_shard_n; else CK(d2h(c.ch_nmax, 0, NCH * 4, v.data()));
      put(v); return SCAN_OK;
    }
    case SCAN_OUT_CL_MISMATCH: {
      const uint64_t ncl = (uint64_t)c.TP * c.PP;
      std::vector<uint32_t> J(ncl), mx(ncl);
      CK(d2h(c.cl_J, 0, ncl * 4, J.data())); CK(d2h(c.cl_max, 0, ncl * 4, mx.data()));
      std::vector<uint8_t> v(ncl, 0);
      if (c.DP >= 2) for (uint64_t i = 0; i < ncl; ++i) v[i] = J[i] != mx[i];
      put(v); return SCAN_OK;
    }
    case SCAN_OUT_LK_WINDOW: case SCAN_OUT_LK_SRC: case SCAN_OUT_LK_DST: {
      std::vector<uint32_t> v((uint64_t)c.NW * np);
      for (uint64_t w = 0; w < c.NW; ++w)
        for (uint64_t l = 0; l < np; ++l)
          v[w * np + l] = which == SCAN_OUT_LK_WINDOW ? (uint32_t)w : (which == SCAN_OUT_LK_SRC ? psrc[l] : pdst[l]);
      put(v); return SCAN_OK;
    }
    case SCAN_OUT_EG_WINDOW: case SCAN_OUT_EG_SRC: case SCAN_OUT_EG_DST: case SCAN_OUT_EG_WEIGHT: {
      const uint64_t W = c.W, nnz_tot = c.nnz_c + W * PCAP;
      std::vector<uint64_t> nbo(W + 1);
      std::vector<uint32_t> nbc(c.nnz_c), nbp(W * PCAP), nbpn(W);
      std::vector<unsigned long long> ew(c.NW * nnz_tot);
      CK(d2h(c.nbc_off, 0, (W + 1) * 8, nbo.data())); CK(d2h(c.nbc, 0, c.nnz_c * 4, nbc.data()));
      CK(d2h(c.nbp, 0, W * PCAP * 4, nbp.data())); CK(d2h(c.nbp_n, 0, W * 4, nbpn.data()));
      CK(d2h(c.ewc, 0, ew.size() * 8, ew.data()));
      std::vector<uint32_t> vw, vs, vd; std::vector<uint64_t> vx;
      for (uint64_t w = 0; w < c.NW; ++w)
        for (uint64_t r = 0; r < W; ++r) {
          std::vector<std::pair<uint32_t, uint64_t>> e;
          for (uint64_t q = nbo[r]; q < nbo[r + 1]; ++q) if (ew[w * nnz_tot + q]) e.push_back({nbc[q], ew[w * nnz_tot + q]});
          for (uint64_t q = 0; q < nbpn[r]; ++q) {
            const uint64_t x = ew[w * nnz_tot + c.nnz_c + r * PCAP + q];
            if (x) e.push_back({nbp[r * PCAP + q], x});
          }
          std::sort(e.begin(), e.end());
          for (size_t i = 0; i < e.size(); ++i) {
            if (i && e[i].first == e[i - 1].first) { vx.back() += e[i].second; continue; }
            vw.push_back((uint32_t)w); vs.push_back((uint32_t)r); vd.push_back(e[i].first); vx.push_back(e[i].second);
          }
        }
      if (which == SCAN_OUT_EG_WINDOW) put(vw); else if (which == SCAN_OUT_EG_SRC) put(vs);
      else if (which == SCAN_OUT_EG_DST) put(vd); else put(vx);
      return SCAN_OK;
    }
    default: return SCAN_E_INVALID_ARG;
  }
}

// direct device arrays: returns buffer + byte range, stage requirement (1 match, 2 detect, 3 localize)
bool direct(Ctx& c, scan_output which, OutDesc& d) {
  const uint64_t W = c.W, items = (uint64_t)c.NW * W, nlk = (uint64_t)c.NW * c.n_p2p, ncl = (uint64_t)c.TP * c.PP;
  switch (which) {
    case SCAN_OUT_RK_SUM_COMPUTE: d = {&c.rk_sum, 0, W * 8, 3}; return true;
    case SCAN_OUT_RK_SUM_WAIT: d = {&c.rk_sum, W * 8, W * 8, 3}; return true;
    case SCAN_OUT_RK_SUM_TRANSFER: d = {&c.rk_sum, 2 * W * 8, W * 8, 3}; return true;
    case SCAN_OUT_CL_J: d = {&c.cl_J, 0, ncl * 4, 2}; return true;
    case SCAN_OUT_WD_TOTAL: d = {&c.wd_total, 0, items * 4, 2}; return true;
    case SCAN_OUT_WD_SLOW: d = {&c.wd_slow, 0, items * 4, 2}; return true;
    case SCAN_OUT_WD_CAND: d = {&c.wd_cand, 0, items, 2}; return true;
    case SCAN_OUT_WD_FRAC: d = {&c.wd_frac, 0, items * 8, 2}; return true;
    case SCAN_OUT_WL_JOINED: d = {&c.wl_joined, 0, items * 4, 3}; return true;
    case SCAN_OUT_WL_LATE: d = {&c.wl_late, 0, items * 4, 3}; return true;
    case SCAN_OUT_WL_LATE_FRAC: d = {&c.wl_frac, 0, items * 8, 3}; return true;
    case SCAN_OUT_WL_VERDICT: d = {&c.wl_verdict, 0, items, 3}; return true;
    case SCAN_OUT_WL_LINK_SLOW: d = {&c.wl_link_slow, 0, items, 3}; return true;
    case SCAN_OUT_LK_N: d = {&c.lk_n, 0, nlk * 4, 3}; return true;
    case SCAN_OUT_LK_MED_PAYLOAD: d = {&c.lk_medp, 0, nlk * 4, 3}; return true;
    case SCAN_OUT_LK_MED_TRANSFER: d = {&c.lk_medt, 0, nlk * 4, 3}; return true;
    case SCAN_OUT_LK_USED_WARM: d = {&c.lk_used, 0, nlk, 3}; return true;
    case SCAN_OUT_LK_SLOW: d = {&c.lk_slow, 0, nlk, 3}; return true;
    case SCAN_OUT_LK_DIR: d = {&c.lk_dir, 0, nlk, 3}; return true;
    case SCAN_OUT_LK_ELIGIBLE: d = {&c.lk_elig, 0, nlk, 3}; return true;
    case SCAN_OUT_LK_MED_BW: d = {&c.lk_bw, 0, nlk * 8, 3}; return true;
    case SCAN_OUT_LB_LABEL: d = {&c.lb_label, 0, items, 3}; return true;
    case SCAN_OUT_LB_ROOT_KIND: d = {&c.lb_rkind, 0, items, 3}; return true;
    case SCAN_OUT_LB_ROOT_RANK: d = {&c.lb_rrank, 0, items * 4, 3}; return true;
    case SCAN_OUT_LB_ROOT_SRC: d = {&c.lb_rsrc, 0, items * 4, 3}; return true;
    case SCAN_OUT_LB_DEPTH: d = {&c.lb_depth, 0, items * 4, 3}; return true;
    case SCAN_OUT_LB_TOTAL_WAIT: d = {&c.lb_twait, 0, items * 8, 3}; return true;
    case SCAN_OUT_COMM_INST: d = {&c.inst_c, 0, c.n_comm * 4, 1}; return true;
    case SCAN_OUT_COMM_WAIT: d = {&c.wait_c, 0, c.n_comm * 4, 3}; return true;
    case SCAN_OUT_SLOW_BITS: d = {&c.bits, 0, c.n_bits_words * 4, 2}; return true;
    case SCAN_OUT_AL_START: d = {&c.al_start, 0, c.aligned ? c.N * 8 : 0, 1}; return true;
    case SCAN_OUT_AL_LEVEL: d = {&c.al_level, 0, c.aligned ? W * 4 : 0, 1}; return true;
    case SCAN_OUT_AL_NANCHOR: d = {&c.al_nanc, 0, c.aligned ? W * 4 : 0, 1}; return true;
    case SCAN_OUT_AL_RESIDUAL: d = {&c.al_resid, 0, c.aligned ? W * 8 : 0, 1}; return true;
    case SCAN_OUT_BL_ROOT: d = {&c.bl_root, 0, c.blamed ? c.N * 8 : 0, 3}; return true;
    case SCAN_OUT_BL_INFLICTED: d = {&c.bl_rank, 0, c.blamed ? W * 8 : 0, 3}; return true;
    case SCAN_OUT_BL_SELF: d = {&c.bl_rank, W * 8, c.blamed ? W * 8 : 0, 3}; return true;
    case SCAN_OUT_BL_UNATTRIBUTED: d = {&c.bl_rank, 2 * W * 8, c.blamed ? W * 8 : 0, 3}; return true;
    case SCAN_OUT_BL_SUFFERED: d = {&c.bl_rank, 3 * W * 8, c.blamed ? W * 8 : 0, 3}; return true;
    default: return false;
  }
}

int stage_of(Ctx& c) { return c.localized ? 3 : c.detected ? 2 : c.matched ? 1 : 0; }

uint64_t ev_bytes(Ctx& c, scan_output w) { return w == SCAN_OUT_EV_SLOW ? c.N : c.N * 4; }
uint64_t in_bytes(Ctx& c, scan_output w) { return w == SCAN_OUT_IN_FLAGS ? c.n_inst : c.n_inst * 4; }

}  // namespace

extern "C" {

static bool stream_output(scan_output which) {  // window-level outputs of a stream context
  return (which >= SCAN_OUT_RK_SUM_COMPUTE && which <= SCAN_OUT_RK_SUM_TRANSFER) ||
         (which >= SCAN_OUT_WD_TOTAL && which <= SCAN_OUT_EG_WEIGHT);
}

scan_status scan_output_size(scan_ctx* ctx, scan_output which, uint64_t* bytes) {
  if (!ctx || !bytes) return SCAN_E_INVALID_ARG;
  Ctx& c = ctx->c;
  *bytes = 0;
  if (c.stream_mode && !stream_output(which)) {
    c.err = "a stream context exports the window-level outputs only (RK_SUM_*, WD_*, WL_*, LK_*, LB_*, EG_*)";
    return SCAN_E_UNSUPPORTED;
  }
  if (!c.matched) return SCAN_OK;
  OutDesc d;
  if (direct(c, which, d)) { if (stage_of(c) >= d.stage) *bytes = d.bytes; return SCAN_OK; }
  if (which <= SCAN_OUT_EV_REF) { *bytes = ev_bytes(c, which); return SCAN_OK; }
  if (which >= SCAN_OUT_IN_CHANNEL && which <= SCAN_OUT_IN_PAYLOAD) { *bytes = in_bytes(c, which); return SCAN_OK; }
  std::vector<uint8_t> t;
  scan_status st = host_table(c, which, t);
  if (st) return st;
  *bytes = t.size();
  return SCAN_OK;
}

scan_status scan_export(scan_ctx* ctx, scan_output which, void* dst, uint64_t dst_bytes, int dst_is_device) {
  if (!ctx) return SCAN_E_INVALID_ARG;
  Ctx& c = ctx->c;
  if (!c.matched) { c.err = "nothing to export before scan_match_collectives"; return SCAN_E_ORDER; }
  CK(cudaSetDevice(c.device));
  const cudaMemcpyKind kind = dst_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  flush_fills(c);
  if (c.stream_mode && !stream_output(which)) {
    c.err = "a stream context exports the window-level outputs only (RK_SUM_*, WD_*, WL_*, LK_*, LB_*, EG_*)";
    return SCAN_E_UNSUPPORTED;
  }
  if (which >= SCAN_OUT_AL_START && which <= SCAN_OUT_AL_RESIDUAL && !c.aligned) { c.err = "scan_align not run"; return SCAN_E_ORDER; }
  if (which >= SCAN_OUT_BL_ROOT && which <= SCAN_OUT_BL_SUFFERED && !c.blamed) { c.err = "scan_blame not run"; return SCAN_E_ORDER; }
  if ((which == SCAN_OUT_COMM_WAIT || which == SCAN_OUT_EV_WAIT) && c.xwait_pending && c.localized) {
    launch_xwait_scatter(c);  // comm-order view of the cross-stage waits (once per analysis)
    CK(cudaStreamSynchronize(c.stream));
    CK(cudaGetLastError());
    c.xwait_pending = false;
  }
  OutDesc d;
  if (direct(c, which, d)) {
    if (stage_of(c) < d.stage) { c.err = "output not computed yet"; return SCAN_E_ORDER; }
    if (dst_bytes < d.bytes) { c.err = "destination too small"; return SCAN_E_INVALID_ARG; }
    if (d.bytes) CK(cudaMemcpyAsync(dst, (const uint8_t*)d.buf->p + d.off_bytes, d.bytes, kind, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    return SCAN_OK;
  }
  const bool ev = which <= SCAN_OUT_EV_REF, in = which >= SCAN_OUT_IN_CHANNEL && which <= SCAN_OUT_IN_PAYLOAD;
  if (ev) {  // fused results: build the general tile prefixes once (untimed)
    scan_status st = ensure_tiles(c);
    if (st) return st;
  }
  if (ev || in) {
    const uint64_t nb = ev ? ev_bytes(c, which) : in_bytes(c, which);
    if (dst_bytes < nb) { c.err = "destination too small"; return SCAN_E_INVALID_ARG; }
    if (!nb) return SCAN_OK;
    void* tgt = dst;
    if (!dst_is_device) { CK(c.scratch.ensure(std::max<size_t>(c.scratch.cap, nb))); tgt = c.scratch.p; }
    if (ev) launch_expand_events(c, which, tgt); else launch_instance_export(c, which, tgt);
    CK(cudaGetLastError());
    if (!dst_is_device) CK(cudaMemcpyAsync(dst, tgt, nb, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    // the walk's scratch lives in c.scratch too: exports after localize may overwrite it, which is fine
    return SCAN_OK;
  }
  std::vector<uint8_t> t;
  scan_status st = host_table(c, which, t);
  if (st) return st;
  if (dst_bytes < t.size()) { c.err = "destination too small"; return SCAN_E_INVALID_ARG; }
  if (!t.empty()) CK(cudaMemcpy(dst, t.data(), t.size(), dst_is_device ? cudaMemcpyHostToDevice : cudaMemcpyHostToHost));
  return SCAN_OK;
}

const void* scan_output_device_ptr(scan_ctx* ctx, scan_output which) {
  if (!ctx) return nullptr;
  Ctx& c = ctx->c;
  OutDesc d;
  if (which != SCAN_OUT_COMM_INST && which != SCAN_OUT_COMM_WAIT && which != SCAN_OUT_SLOW_BITS) return nullptr;
  if (!direct(c, which, d) || stage_of(c) < d.stage) return nullptr;
  flush_fills(c);
  if (which == SCAN_OUT_COMM_WAIT && c.xwait_pending) {
    launch_xwait_scatter(c);
    if (cudaStreamSynchronize(c.stream) != cudaSuccess) return nullptr;
    c.xwait_pending = false;
  }
  return (const uint8_t*)d.buf->p + d.off_bytes;
}

}  // extern "C"
