// stream.cu — NEXT-3: sliding-window streaming ("on-line" analysis; SURVEY.md §8(f)
// rank 3; the C5 workload re-analyses the last K iterations after every new one).
//
// The window result equals scan_analyze on the window's events (one window): instances never
// straddle iterations (reading R30), so every per-rank / per-edge quantity is a sum of
// per-iteration partials, the stage-2 segments that cross an iteration boundary are fixed up from
// per-rank boundary records (as between shards, shard.cu), and the stage-3 link medians are taken
// over the window's samples. Each push therefore analyses ONE iteration (the fused pass on a
// sub-context, stopped before candidates / links / walk), snapshots its partials into ring slot
// pushes % K, and recombines the window on the device:
//   k_stream_pack    P2P samples of the iteration (transfer, payload, flags) into its ring slot
//   k_stream_sum     per-rank counters, wait-for edge weights, per-rank sums over the window
//   k_stream_ht      stage-2 boundary records in age order -> k_shard_fixup
//   k_stream_window  window samples link-major, age-minor (= the window's instance order, so the
//                    median's tie-break is the from-scratch one) -> k_link_median, k_link_flags
//   then candidates, verdicts and the walk.
// Requirements: every pushed iteration is SPMD (fused path) with the same channel structure as the
// first one (per-link instance counts); the window is a single window (window_iters of the
// analysis = 0). Only the window-level outputs (WD_*, WL_*, LK_*, LB_*, EG_*, RK_SUM_*) exist.
#include <algorithm>
#include <array>
#include <cstring>
#include <sstream>
#include "internal.cuh"

namespace ms {

struct StreamState {
  scan_topology topo{};
  std::vector<uint64_t> coff;
  std::vector<uint32_t> cmem;
  uint32_t K = 0;
  uint64_t pushes = 0;
  scan_ctx* sub = nullptr;
  bool ready = false;
  uint64_t nnz_tot = 0, npi = 0;
  uint32_t np = 0;
  std::vector<uint32_t> nl, loff;  // per link: instances per iteration, offset in an iteration block
  std::vector<std::array<uint64_t, 4>> cnt;  // per slot: incomplete, kind / payload mismatch, instances
  DevBuf rg_w32, rg_ew, rg_rk, rg_ht, rg_smp, d_nl, d_loff, d_slots, ht_age;
  DevBuf w_base, w_slot, w_nmax, w_rec, w_pay, w_iter, w_key;
};

namespace {

__global__ void k_stream_pack(uint32_t n_comms, const uint32_t* nl, const uint32_t* loff, const uint64_t* ch_base,
                              const uint64_t* ch_slot, const uint4* rec, const uint4* slots, uint32_t* out) {
  const uint32_t l = blockIdx.x;
  const uint64_t b = ch_base[n_comms + l], sb = ch_slot[n_comms + l];
  for (uint32_t k = threadIdx.x; k < nl[l]; k += blockDim.x) {
    const uint4 r = rec[b + k];
    uint32_t* o = out + 3ull * (loff[l] + k);
    o[0] = r.x;
    o[1] = (r.w & SCAN_F_VALID) ? slots[sb + 2ull * k].w : 0u;  // the send slot's payload (valid samples only)
    o[2] = r.w & 0xFFu;
  }
}

__global__ void k_stream_sum(uint32_t Kv, const uint32_t* slots, uint64_t W, uint64_t nnz, const uint32_t* rg_w32,
                             const unsigned long long* rg_ew, const unsigned long long* rg_rk, uint32_t* wd_total,
                             uint32_t* wd_slow, uint32_t* wl_joined, uint32_t* wl_late, unsigned long long* ew,
                             unsigned long long* rk) {
  const uint64_t n32 = 4 * W, tot = n32 + nnz + 3 * W;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (uint64_t)gridDim.x * blockDim.x) {
    if (i < n32) {
      uint32_t v = 0;
      for (uint32_t a = 0; a < Kv; ++a) v += rg_w32[(uint64_t)slots[a] * n32 + i];
      const uint64_t sec = i / W, j = i - sec * W;
      uint32_t* dst = sec == 0 ? wd_total : sec == 1 ? wd_slow : sec == 2 ? wl_joined : wl_late;
      dst[j] = v;
    } else if (i < n32 + nnz) {
      const uint64_t j = i - n32;
      unsigned long long v = 0;
      for (uint32_t a = 0; a < Kv; ++a) v += rg_ew[(uint64_t)slots[a] * nnz + j];
      ew[j] = v;
    } else {
      const uint64_t j = i - n32 - nnz;
      unsigned long long v = 0;
      for (uint32_t a = 0; a < Kv; ++a) v += rg_rk[(uint64_t)slots[a] * 3 * W + j];
      rk[j] = v;
    }
  }
}

__global__ void k_stream_ht(uint32_t Kv, const uint32_t* slots, uint64_t W, const unsigned long long* rg_ht,
                            unsigned long long* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < Kv * W; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = i / W, r = i - a * W;
    out[i] = rg_ht[(uint64_t)slots[a] * W + r];
  }
}

// window samples of link l, age a, occurrence k at Kv * loff[l] + a * nl[l] + k
__global__ void k_stream_window(uint32_t Kv, const uint32_t* slots, uint64_t npi, const uint32_t* nl, const uint32_t* loff,
                                const uint32_t* rg_smp, uint4* w_rec, uint32_t* w_pay, unsigned long long* w_key) {
  const uint32_t l = blockIdx.x, a = blockIdx.y;
  const uint64_t src0 = (uint64_t)slots[a] * npi + loff[l], dst0 = (uint64_t)Kv * loff[l] + (uint64_t)a * nl[l];
  for (uint32_t k = threadIdx.x; k < nl[l]; k += blockDim.x) {
    const uint32_t* v = rg_smp + 3 * (src0 + k);
    w_rec[dst0 + k] = make_uint4(v[0], 0u, 0u, v[2]);
    w_pay[2 * (dst0 + k)] = v[1];
    w_pay[2 * (dst0 + k) + 1] = 0u;
    w_key[dst0 + k] = lk_sample_key(v[2], v[0], v[1]);
  }
}

StreamState* state(Ctx& c) { return static_cast<StreamState*>(c.stream_state); }

// window-level structure (tables the combine / median / walk read) from the first analysed iteration
scan_status establish(Ctx& c, StreamState& S, Ctx& u) {
  c.TP = u.TP; c.PP = u.PP; c.DP = u.DP; c.W = u.W; c.n_comms = u.n_comms; c.NW = 1;
  c.n_p2p = u.n_p2p; c.NCH = u.n_comms + u.n_p2p; c.nnz_c = u.nnz_c; c.n_bits_words = 1; c.n_comp = 0;
  S.np = (uint32_t)u.n_p2p;
  S.nnz_tot = u.nnz_c + (uint64_t)u.W * PCAP;
  const uint64_t W = c.W;
  CK(c.nbc_off.ensure((W + 1) * 8)); CK(c.nbc.ensure(std::max<uint64_t>(c.nnz_c, 1) * 4));
  CK(c.nbp.ensure(W * PCAP * 4)); CK(c.nbp_n.ensure(W * 4));
  CK(c.ch_nsend.ensure(std::max<uint64_t>(2ull * S.np, 1) * 4)); CK(c.ch_nrecv.ensure(std::max<uint64_t>(2ull * S.np, 1) * 4));
  const cudaMemcpyKind dd = cudaMemcpyDeviceToDevice;
  CK(cudaMemcpyAsync(c.nbc_off.p, u.nbc_off.p, (W + 1) * 8, dd, c.stream));
  if (c.nnz_c) CK(cudaMemcpyAsync(c.nbc.p, u.nbc.p, c.nnz_c * 4, dd, c.stream));
  CK(cudaMemcpyAsync(c.nbp.p, u.nbp.p, W * PCAP * 4, dd, c.stream));
  CK(cudaMemcpyAsync(c.nbp_n.p, u.nbp_n.p, W * 4, dd, c.stream));
  if (S.np) {
    CK(cudaMemcpyAsync(c.ch_nsend.as<uint32_t>() + S.np, u.ch_nsend.as<uint32_t>() + S.np, S.np * 4ull, dd, c.stream));
    CK(cudaMemcpyAsync(c.ch_nrecv.as<uint32_t>() + S.np, u.ch_nrecv.as<uint32_t>() + S.np, S.np * 4ull, dd, c.stream));
  }
  S.nl.assign(S.np, 0);
  if (S.np) CK(cudaMemcpy(S.nl.data(), u.ch_nmax.as<uint32_t>() + u.n_comms, S.np * 4ull, cudaMemcpyDeviceToHost));
  S.loff.assign(S.np + 1, 0);
  for (uint32_t l = 0; l < S.np; ++l) S.loff[l + 1] = S.loff[l] + S.nl[l];
  S.npi = S.loff[S.np];
  scan_status st;
  if ((st = upload(c, S.d_nl, S.nl)) || (st = upload(c, S.d_loff, S.loff))) return st;
  const uint64_t K = S.K;
  CK(S.rg_w32.ensure(K * 4 * W * 4)); CK(S.rg_ew.ensure(K * S.nnz_tot * 8)); CK(S.rg_rk.ensure(K * 3 * W * 8));
  CK(S.rg_ht.ensure(K * W * 8)); CK(S.ht_age.ensure(K * W * 8)); CK(S.rg_smp.ensure(std::max<uint64_t>(K * S.npi * 12, 16)));
  CK(S.d_slots.ensure(K * 4));
  CK(S.w_base.ensure((c.NCH + 1) * 8)); CK(S.w_slot.ensure((c.NCH + 1) * 8)); CK(S.w_nmax.ensure((c.NCH + 1) * 4));
  CK(S.w_rec.ensure(std::max<uint64_t>(K * S.npi * 16, 16))); CK(S.w_pay.ensure(std::max<uint64_t>(K * S.npi * 8, 16)));
  CK(S.w_iter.ensure(std::max<uint64_t>(K * S.npi * 4, 16))); CK(S.w_key.ensure(std::max<uint64_t>(K * S.npi * 8, 16)));
  CK(cudaMemsetAsync(S.w_iter.p, 0, std::max<uint64_t>(K * S.npi * 4, 16), c.stream));
  S.cnt.assign(K, {0, 0, 0, 0});
  if ((st = alloc_detect(c)) || (st = alloc_localize(c))) return st;
  flush_fills(c);  // the zero fills of the window buffers run before the first combine writes them
  S.ready = true;
  return SCAN_OK;
}

}  // namespace

void stream_release(Ctx& c) {
  StreamState* S = state(c);
  if (!S) return;
  if (S->sub) scan_destroy(S->sub);
  for (DevBuf* b : {&S->rg_w32, &S->rg_ew, &S->rg_rk, &S->rg_ht, &S->rg_smp, &S->d_nl, &S->d_loff, &S->d_slots, &S->ht_age,
                    &S->w_base, &S->w_slot, &S->w_nmax, &S->w_rec, &S->w_pay, &S->w_iter, &S->w_key})
    b->release();
  delete S;
  c.stream_state = nullptr;
}

}  // namespace ms

using namespace ms;

extern "C" {

scan_status scan_stream_open(scan_ctx* ctx, const scan_topology* topo, const scan_comm_table* comms, uint32_t window_iters,
                             const scan_detect_config* dcfg, const scan_localize_config* lcfg) {
  if (!ctx || !topo || !comms || window_iters == 0 || window_iters > 4096) return SCAN_E_INVALID_ARG;
  if (comms->n_comms && (!comms->offsets || !comms->members)) return SCAN_E_INVALID_ARG;
  Ctx& c = ctx->c;
  if (c.n_shards > 1) { c.err = "streaming on a sharded context is not supported"; return SCAN_E_UNSUPPORTED; }
  stream_release(c);
  StreamState* S = new StreamState();
  c.stream_state = S;
  S->topo = *topo;
  if (comms->n_comms) S->coff.assign(comms->offsets, comms->offsets + comms->n_comms + 1);
  else S->coff.assign(1, 0);  // n_comms == 0 accepts offsets == NULL
  S->cmem.assign(comms->members, comms->members + S->coff.back());
  S->K = window_iters;
  scan_status st = scan_create(&S->sub, c.device, c.stream);
  if (st) { c.err = "streaming: sub-context creation failed"; return st; }
  c.dcfg = dcfg ? *dcfg : scan_detect_config{3, 2, 50000, 3, 10, 10, 0, 0, 0};
  c.lcfg = lcfg ? *lcfg : scan_localize_config{100000, 7, 10, 7, 10, 10, 3, 0, 0, 100000};
  c.dcfg.window_iters = 0;  // the window is one analysis window
  c.loaded = c.matched = c.detected = c.localized = false;
  c.stream_mode = true;
  return SCAN_OK;
}

scan_status scan_stream_push(scan_ctx* ctx, const scan_event_columns* iteration, uint32_t flags, scan_localize_result* out) {
  if (!ctx || !iteration) return SCAN_E_INVALID_ARG;
  Ctx& c = ctx->c;
  StreamState* Sp = state(c);
  if (!Sp) { c.err = "scan_stream_push before scan_stream_open"; return SCAN_E_ORDER; }
  StreamState& S = *Sp;
  CK(cudaSetDevice(c.device));
  Ctx& u = S.sub->c;
  // 1. the new iteration, analysed alone (fused pass, partials only)
  scan_status st;
  const uint64_t W0 = (uint64_t)S.topo.tp * S.topo.pp * S.topo.dp;
  bool same = S.ready && iteration->rank_offsets && u.h_rank_off.size() == W0 + 1 &&
              std::equal(u.h_rank_off.begin(), u.h_rank_off.end(), iteration->rank_offsets);
  if (same) {  // same per-rank counts as the previous iteration: new columns, cached structure
    const uint64_t N = u.N;
    if (flags & SCAN_DEVICE_PTRS) {
      const void* ptrs[] = {iteration->dur_ns, iteration->kind_op, iteration->meta, iteration->comm, iteration->payload_bytes};
      for (const void* p : ptrs)
        if (N && ((uintptr_t)p & 15)) { c.err = "device columns must be 16-byte aligned"; return SCAN_E_INVALID_ARG; }
      u.d_dur = iteration->dur_ns; u.d_kind = iteration->kind_op; u.d_meta = iteration->meta;
      u.d_comm = iteration->comm; u.d_pay = iteration->payload_bytes;
    } else {
      CK(u.own_dur.ensure(N * 4)); CK(u.own_kind.ensure(N * 2)); CK(u.own_meta.ensure(N * 2));
      CK(u.own_comm.ensure(N * 4)); CK(u.own_pay.ensure(N * 4));
      const cudaMemcpyKind hd = cudaMemcpyHostToDevice;
      CK(cudaMemcpyAsync(u.own_dur.p, iteration->dur_ns, N * 4, hd, u.stream));
      CK(cudaMemcpyAsync(u.own_kind.p, iteration->kind_op, N * 2, hd, u.stream));
      CK(cudaMemcpyAsync(u.own_meta.p, iteration->meta, N * 2, hd, u.stream));
      CK(cudaMemcpyAsync(u.own_comm.p, iteration->comm, N * 4, hd, u.stream));
      CK(cudaMemcpyAsync(u.own_pay.p, iteration->payload_bytes, N * 4, hd, u.stream));
      u.d_dur = u.own_dur.as<uint32_t>(); u.d_kind = u.own_kind.as<uint16_t>(); u.d_meta = u.own_meta.as<uint16_t>();
      u.d_comm = u.own_comm.as<uint32_t>(); u.d_pay = u.own_pay.as<uint32_t>();
    }
    if ((st = fused_rerun(u))) { c.err = std::string("streaming analysis: ") + u.err; return st; }
  } else {
    scan_comm_table ct{(uint32_t)(S.coff.size() - 1), S.coff.data(), S.cmem.data()};
    st = scan_load_events(S.sub, &S.topo, &ct, iteration, flags & (SCAN_HOST_PTRS | SCAN_DEVICE_PTRS));
    if (st) { c.err = std::string("streaming load: ") + u.err; return st; }
    if (!u.spmd) { c.err = "streaming needs SPMD iterations"; return SCAN_E_UNSUPPORTED; }
    u.dcfg = c.dcfg; u.lcfg = c.lcfg; u.partial_tail = true;
    if ((st = fused_all(u))) { c.err = std::string("streaming analysis: ") + u.err; return st < 0 ? st : SCAN_E_UNSUPPORTED; }
  }
  if (!S.ready) {
    if ((st = establish(c, S, u))) return st;
  } else if (!same) {  // a reloaded iteration: its channel structure must be the first one's
    std::vector<uint32_t> nl(S.np);
    bool ok = u.n_p2p == S.np && u.W == c.W && u.nnz_c == c.nnz_c;
    if (ok && S.np) {
      CK(cudaMemcpy(nl.data(), u.ch_nmax.as<uint32_t>() + u.n_comms, S.np * 4ull, cudaMemcpyDeviceToHost));
      ok = nl == S.nl;
    }
    if (!ok) { c.err = "streaming: an iteration's channel structure differs from the first one"; return SCAN_E_UNSUPPORTED; }
  }
  const uint64_t W = c.W, K = S.K, s = S.pushes % K;
  // 2. snapshot the iteration's partials into ring slot s
  const cudaMemcpyKind dd = cudaMemcpyDeviceToDevice;
  uint32_t* w32 = S.rg_w32.as<uint32_t>() + s * 4 * W;
  CK(cudaMemcpyAsync(w32, u.wd_total.p, W * 4, dd, c.stream));
  CK(cudaMemcpyAsync(w32 + W, u.wd_slow.p, W * 4, dd, c.stream));
  CK(cudaMemcpyAsync(w32 + 2 * W, u.wl_joined.p, W * 4, dd, c.stream));
  CK(cudaMemcpyAsync(w32 + 3 * W, u.wl_late.p, W * 4, dd, c.stream));
  CK(cudaMemcpyAsync(S.rg_ew.as<unsigned long long>() + s * S.nnz_tot, u.ewc.p, S.nnz_tot * 8, dd, c.stream));
  CK(cudaMemcpyAsync(S.rg_rk.as<unsigned long long>() + s * 3 * W, u.rk_sum.p, 3 * W * 8, dd, c.stream));
  c.launches += launch_shard_head(u, S.rg_ht.as<unsigned long long>() + s * W);
  if (S.np) {
    k_stream_pack<<<S.np, 128, 0, c.stream>>>(u.n_comms, S.d_nl.as<uint32_t>(), S.d_loff.as<uint32_t>(), u.ch_base.as<uint64_t>(),
                                             u.ch_slot.as<uint64_t>(), u.inst_rec.as<uint4>(), u.slots.as<uint4>(),
                                             S.rg_smp.as<uint32_t>() + 3 * s * S.npi);
    c.launches += 1;
  }
  S.cnt[s] = {u.hc.n_incomplete, u.hc.n_kind_mismatch, u.hc.n_payload_mismatch, u.n_inst};
  S.pushes += 1;
  // 3. the window: age-ordered slots, sums, stage-2 boundary fix-up, window samples
  const uint32_t Kv = (uint32_t)std::min<uint64_t>(S.pushes, K);
  std::vector<uint32_t> slots(Kv);
  for (uint32_t a = 0; a < Kv; ++a) slots[a] = (uint32_t)((S.pushes - Kv + a) % K);
  if ((st = upload(c, S.d_slots, slots))) return st;
  const uint64_t tot = 7 * W + S.nnz_tot;
  flush_fills(c);
  k_stream_sum<<<(unsigned)std::min<uint64_t>((tot + 255) / 256, 2048), 256, 0, c.stream>>>(
      Kv, S.d_slots.as<uint32_t>(), W, S.nnz_tot, S.rg_w32.as<uint32_t>(), S.rg_ew.as<unsigned long long>(),
      S.rg_rk.as<unsigned long long>(), c.wd_total.as<uint32_t>(), c.wd_slow.as<uint32_t>(), c.wl_joined.as<uint32_t>(),
      c.wl_late.as<uint32_t>(), c.ewc.as<unsigned long long>(), c.rk_sum.as<unsigned long long>());
  c.launches += 1;
  if (c.lcfg.stage2_mode == 0 && Kv > 1) {
    k_stream_ht<<<(unsigned)std::min<uint64_t>((Kv * W + 255) / 256, 2048), 256, 0, c.stream>>>(
        Kv, S.d_slots.as<uint32_t>(), W, S.rg_ht.as<unsigned long long>(), S.ht_age.as<unsigned long long>());
    c.launches += 1 + launch_shard_fixup(c, (int)Kv, S.ht_age.as<unsigned long long>());
  }
  if (S.np) {
    std::vector<uint64_t> wb(c.NCH + 1, 0), ws(c.NCH + 1, 0);
    std::vector<uint32_t> wn(c.NCH + 1, 0);
    for (uint32_t l = 0; l < S.np; ++l) {
      wb[c.n_comms + l] = (uint64_t)Kv * S.loff[l];
      ws[c.n_comms + l] = 2ull * Kv * S.loff[l];
      wn[c.n_comms + l] = Kv * S.nl[l];
    }
    if ((st = upload(c, S.w_base, wb)) || (st = upload(c, S.w_slot, ws)) || (st = upload(c, S.w_nmax, wn))) return st;
    k_stream_window<<<dim3(S.np, Kv), 128, 0, c.stream>>>(Kv, S.d_slots.as<uint32_t>(), S.npi, S.d_nl.as<uint32_t>(),
                                                         S.d_loff.as<uint32_t>(), S.rg_smp.as<uint32_t>(), S.w_rec.as<uint4>(),
                                                         S.w_pay.as<uint32_t>(), S.w_key.as<unsigned long long>());
    c.launches += 1;
  }
  // 4. candidates, links, verdicts and the walk on the window
  {
    Counters z{};
    z.bad_event = ~0ull;
    CK(cudaMemcpyAsync(c.counters.p, &z, sizeof(Counters), cudaMemcpyHostToDevice, c.stream));
  }
  CK(cudaMemsetAsync(c.wl_link_slow.p, 0, W, c.stream));
  CK(cudaMemsetAsync(c.lk_slow.p, 0, (uint64_t)S.np + 1, c.stream));
  CK(cudaMemsetAsync(c.scratch.as<uint32_t>() + 2 * W, 0, (c.NW + 2) * 4, c.stream));
  c.launches += timed(c, "k_wd_finish", [&] { return launch_wd_finish(c); });
  c.launches += timed(c, "k_link_median", [&] {
    return launch_link_median_window(c, S.w_base.as<uint64_t>(), S.w_nmax.as<uint32_t>(), S.w_slot.as<uint64_t>(),
                                     S.w_rec.as<uint4>(), S.w_iter.as<uint32_t>(), S.w_pay.as<uint32_t>(),
                                     S.w_key.as<unsigned long long>(), (uint64_t)Kv * S.npi);
  });
  c.launches += timed(c, "k_link_flags", [&] { return launch_link_flags(c); });
  c.launches += timed(c, "k_walk", [&] { return launch_verdict_walk(c); });
  if ((st = sync_read(c))) return st;
  if (c.hc.overflow & 24u) { c.err = "capacity exceeded: more than 16384 samples on a link / links in a direction class"; return SCAN_E_UNSUPPORTED; }
  c.matched = c.detected = c.localized = true;
  c.loaded = true;
  uint64_t inc = 0, kmis = 0, pmis = 0;
  for (uint32_t a = 0; a < Kv; ++a) { inc += S.cnt[slots[a]][0]; kmis += S.cnt[slots[a]][1]; pmis += S.cnt[slots[a]][2]; }
  if (out) {
    out->n_windows = 1; out->n_links = S.np; out->n_link_slow = c.hc.n_link_slow;
    out->n_compute_slow = c.hc.v_count[SCAN_V_COMPUTE_SLOW]; out->n_link_slow_ranks = c.hc.v_count[SCAN_V_LINK_SLOW];
    out->n_both = c.hc.v_count[SCAN_V_BOTH]; out->n_exonerated = c.hc.v_count[SCAN_V_EXONERATED];
    out->n_insufficient = c.hc.v_count[SCAN_V_INSUFFICIENT]; out->n_roots = c.hc.n_roots;
    out->n_victims = c.hc.n_victims; out->n_unattributed = c.hc.n_unattributed; out->n_edges = 0;
  }
  return (inc || kmis || pmis) ? SCAN_PARTIAL : SCAN_OK;
}

uint64_t scan_stream_window(const scan_ctx* ctx) {
  if (!ctx || !ctx->c.stream_state) return 0;
  const StreamState* S = static_cast<const StreamState*>(ctx->c.stream_state);
  return std::min<uint64_t>(S->pushes, S->K);
}

}  // extern "C"
