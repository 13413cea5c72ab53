// shard.cu — multi-GPU analysis over iteration-window shards.
//
// Shard g of G holds every rank's events for a block of whole iterations (the paper's tracer
// records per-iteration step events; no instance straddles an iteration). The fused
// K9 pass runs unchanged on each shard; four exchanges over NCCL make the results job-wide and
// identical to the unsharded run:
//   X1 ncclAllGather  per-comm member-count extremes, P2P channel bitmap, iteration counts
//   X2 ncclAllGather  per-P2P-channel send / recv counts (P2P channel ids need the OR'ed bitmap)
//      => host: job-wide channel bases / slots (the unsharded k_channels numbering) and this
//         shard's first occurrence per channel `pre`; the shard's kernels get base + pre and
//         slot + pre*|M|, so every instance id / slot they write is the job-wide one
//   X3 grouped ncclSend/ncclRecv  the 12-byte record of each P2P instance to the shard owning
//      its link (pid % G), which then holds every sample of the link for the stage-3 median
//   X4 grouped ncclAllReduce(sum)  per-(window, rank) stage-1/2 counters, wait-for edge weights,
//      per-rank sums, link medians (zero on non-owners), per-rank stage-2 boundary records
//   => every shard: stage-2 boundary fix-up, candidates, LinkSlow flags, verdicts + walk
//      (replicated on identical inputs, so every shard reports the same job-wide tables).
// Exchange volume on C3 at G = 8: X3 ~ 12 B x 14.5e6 P2P instances x 7/8 spread over 8 GPUs;
// X4 ~ 0.6 MB. The per-shard fused pass dominates.
#include <nccl.h>
#include <algorithm>
#include <cstring>
#include <sstream>
#include "internal.cuh"

namespace ms {
namespace {

#define NCK(x)                                                                           \
  do {                                                                                   \
    ncclResult_t _r = (x);                                                               \
    if (_r != ncclSuccess) {                                                             \
      c.err = std::string("NCCL error: ") + ncclGetErrorString(_r) + " at " #x;          \
      return SCAN_E_NCCL;                                                                \
    }                                                                                    \
  } while (0)

// u32 words per shipped P2P instance: what the stage-3 median reads (k_link_median): transfer time
// (rec.x = dmin), payload, and iteration << 8 | instance flags (VALID, WARMUP; P2P class bits are 0)
constexpr uint32_t LREC = 3;

struct LinkMap { unsigned long long flat, inst0, slot0; uint32_t n, pad; };

// X3 pack / unpack: one CTA per (link, shard range); instance k of the range at flat + k
__global__ void k_link_pack(const LinkMap* map, const uint4* rec, const uint32_t* p2p_iter, const uint32_t* p2p_pay,
                            uint64_t p2p_inst0, uint64_t p2p_slot0, uint32_t* buf) {
  const LinkMap m = map[blockIdx.x];
  for (uint32_t k = threadIdx.x; k < m.n; k += blockDim.x) {
    const uint64_t i = m.inst0 + k;
    const uint4 r = rec[i];
    uint32_t* o = buf + (m.flat + k) * LREC;
    o[0] = r.x;
    o[1] = p2p_pay[m.slot0 + 2ull * k - p2p_slot0];
    o[2] = (p2p_iter[i - p2p_inst0] << 8) | (r.w & 0xFFu);
  }
}

// rows of links this shard owns; only the fields the median reads are written (the rest of an
// unowned-range row stays unspecified, scan.h)
__global__ void k_link_unpack(const LinkMap* map, const uint32_t* buf, uint4* rec, uint32_t* p2p_iter, uint32_t* p2p_pay,
                              uint64_t p2p_inst0, uint64_t p2p_slot0) {
  const LinkMap m = map[blockIdx.x];
  for (uint32_t k = threadIdx.x; k < m.n; k += blockDim.x) {
    const uint64_t i = m.inst0 + k;
    const uint32_t* v = buf + (m.flat + k) * LREC;
    rec[i].x = v[0];
    rec[i].w = v[2] & 0xFFu;
    p2p_pay[m.slot0 + 2ull * k - p2p_slot0] = v[1];
    p2p_iter[i - p2p_inst0] = v[2] >> 8;
  }
}

__device__ __forceinline__ bool bits_any_range(const uint32_t* b, uint32_t lo, uint32_t hi) {
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

// Stage-2 boundary record of each rank (reading R11: pslow = the preceding compute segment holds
// a stage-1 slow op; the segment of a shard's first comm event may start in an earlier shard).
// One warp per rank: bit0 has a comm event, bit1 slow op before the first comm event, bit2 that
// event's instance counts for stage 2, bit3 this rank is its unique late last arriver, bit4 slow
// op after the last comm event (all compute events if none), bits 32.. window of that event.
__global__ void k_shard_head(int W, const uint64_t* rank_off, const uint16_t* kind, const uint64_t* comm_off,
                             const uint64_t* bits_off, const uint32_t* r_ncomp, const uint32_t* bits, const uint32_t* inst_c,
                             const uint4* rec, uint32_t classes, unsigned long long late_margin, uint32_t wi,
                             uint32_t it_off, unsigned long long* out) {
  const uint32_t r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= (uint32_t)W) return;
  const uint32_t lane = lane_id();
  const uint64_t e0 = rank_off[r], e1 = rank_off[r + 1];
  uint32_t nc0 = 0, ie0 = 0;
  bool has = false;
  for (uint64_t b = e0; b < e1; b += 32) {  // forward to the first comm event
    const uint64_t e = b + lane;
    const bool in = e < e1;
    const uint32_t kd = in ? kind[e] : 0u;
    const unsigned mc = __ballot_sync(0xFFFFFFFFu, in && (kd & 7u));
    const unsigned mp = __ballot_sync(0xFFFFFFFFu, in && !(kd & 7u));
    const unsigned mi = __ballot_sync(0xFFFFFFFFu, in && (kd & 8u));
    if (mc) {
      const unsigned below = (1u << (__ffs(mc) - 1)) - 1u;
      nc0 += __popc(mp & below); ie0 += __popc(mi & below); has = true;
      break;
    }
    nc0 += __popc(mp); ie0 += __popc(mi);
  }
  const uint32_t ncomp = r_ncomp[r];
  uint32_t nct = ncomp;
  if (has) {  // backward to the last comm event (lane 0 = latest event of the chunk)
    nct = 0;
    uint64_t t = e1;
    while (t > e0) {
      const bool in = (uint64_t)lane < t - e0;
      const uint32_t kd = in ? kind[t - 1 - lane] : 0u;
      const unsigned mc = __ballot_sync(0xFFFFFFFFu, in && (kd & 7u));
      const unsigned mp = __ballot_sync(0xFFFFFFFFu, in && !(kd & 7u));
      if (mc) { nct += __popc(mp & ((1u << (__ffs(mc) - 1)) - 1u)); break; }
      nct += __popc(mp);
      t = t - e0 > 32 ? t - 32 : e0;
    }
  }
  if (lane) return;
  const uint32_t* b = bits + bits_off[r];
  unsigned long long v = (has ? 1ull : 0ull) | (bits_any_range(b, 0, nc0) ? 2ull : 0ull) |
                         (bits_any_range(b, ncomp - nct, ncomp) ? 16ull : 0ull);
  if (has) {
    const uint4 rc = rec[inst_c[comm_off[r]]];
    const uint32_t cls = (rc.w >> 8) & 0xFFu;
    const bool elig = (rc.w & SCAN_F_VALID) && cls && ((classes >> (cls - 1)) & 1u);
    const bool late = (rc.w & SCAN_F_UNIQUE_LAST) && rc.z == r && (unsigned long long)(rc.y - rc.x) > late_margin;
    v |= (elig ? 4ull : 0ull) | (late ? 8ull : 0ull) | ((unsigned long long)(wi ? (it_off + ie0) / wi : 0u) << 32);
  }
  out[r] = v;
}

// Replicated after X4: a shard's first comm event whose segment had no slow op locally joins the
// stage-2 count when the segment's earlier part (previous shards, back to the last comm event)
// held one.
__global__ void k_shard_fixup(int W, int G, const unsigned long long* ht, uint32_t* wl_joined, uint32_t* wl_late) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (uint32_t)W) return;
  for (int s = 1; s < G; ++s) {
    const unsigned long long h = ht[(uint64_t)s * W + r];
    if ((h & 7ull) != 5ull) continue;  // has comm, no local slow op before it, stage-2 eligible
    bool inc = false;
    for (int q = s - 1; q >= 0; --q) {
      const unsigned long long x = ht[(uint64_t)q * W + r];
      if (x & 16ull) { inc = true; break; }
      if (x & 1ull) break;
    }
    if (!inc) continue;
    const uint64_t o = (uint64_t)(h >> 32) * W + r;
    wl_joined[o] += 1;
    if (h & 8ull) wl_late[o] += 1;
  }
}

// X1 send buffer, packed on the device: header from the census counters, per-comm member-count
// extremes, P2P channel bitmap words
__global__ void k_x1_pack(const Counters* cnt, uint32_t force_status, unsigned long long N, const uint32_t* nmin,
                          const uint32_t* nmax, const uint32_t* bitmap, uint32_t nc, uint64_t nbm, uint32_t* out) {
  const uint64_t L = 16 + 2ull * nc + nbm;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    if (i < 16) {
      const unsigned long long be = cnt->bad_event;
      switch ((int)i) {
        case 0: v = force_status ? force_status : (cnt->overflow & NOT_SPMD) ? 1u : be != ~0ull ? 2u : (cnt->overflow & 7u) ? 3u : 0u; break;
        case 1: v = cnt->max_niter; break;
        case 2: v = cnt->min_niter; break;
        case 3: v = cnt->n_end_ranks; break;
        case 4: v = cnt->n_iters; break;
        case 5: v = (uint32_t)N; break;
        case 6: v = (uint32_t)(N >> 32); break;
        case 7: v = (uint32_t)be; break;
        case 8: v = (uint32_t)(be >> 32); break;
        case 9: v = (uint32_t)cnt->n_comm; break;
        case 10: v = (uint32_t)(cnt->n_comm >> 32); break;
        case 11: v = (uint32_t)cnt->n_comp; break;
        case 12: v = (uint32_t)(cnt->n_comp >> 32); break;
        case 13: v = cnt->max_ncomp; break;
        case 14: v = (uint32_t)cnt->n_bits_words; break;
        default: v = (uint32_t)(cnt->n_bits_words >> 32); break;
      }
    } else if (i < 16 + nc) {
      v = nmin[i - 16];
    } else if (i < 16 + 2ull * nc) {
      v = nmax[i - 16 - nc];
    } else {
      v = bitmap[i - 16 - 2ull * nc];
    }
    out[i] = v;
  }
}

// status + match counters of this shard for the X4 all-reduce (no host round trip)
__global__ void k_x4_status(const Counters* cnt, const uint32_t* cl_J, const uint32_t* cl_max, uint32_t ncl, int check_class,
                            unsigned long long* e) {
  if (threadIdx.x || blockIdx.x) return;
  unsigned long long bad = 0;
  if (check_class)
    for (uint32_t i = 0; i < ncl; ++i) bad |= cl_J[i] != cl_max[i];
  e[0] = (cnt->overflow & NOT_SPMD) ? 1ull : 0ull;
  e[1] = bad;
  e[2] = cnt->n_incomplete; e[3] = cnt->n_kind_mismatch; e[4] = cnt->n_payload_mismatch;
}

// all-gather of n u32 already packed in c.x_send; the gathered words land on the host
scan_status allgather_dev(Ctx& c, size_t n, std::vector<uint32_t>& all) {
  const size_t G = (size_t)c.n_shards;
  CK(c.x_recv.ensure(n * 4 * G));
  NCK(ncclAllGather(c.x_send.p, c.x_recv.p, n, ncclUint32, (ncclComm_t)c.nccl, c.stream));
  all.assign(n * G, 0);
  CK(cudaMemcpyAsync(all.data(), c.x_recv.p, n * 4 * G, cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  return SCAN_OK;
}

}  // namespace

scan_status sharded_all(Ctx& c) {
  c.matched = c.detected = c.localized = false;
  c.fused_used = false; c.tiles_ready = false; c.xwait_pending = false;
  const uint32_t G = (uint32_t)c.n_shards, g = (uint32_t)c.shard, nc = c.n_comms;
  const uint64_t W = c.W;
  ncclComm_t comm = (ncclComm_t)c.nccl;
  scan_status st;
  if ((st = prep_ws(c, false))) return st;
  // ---- local census (the fused pre-pass of this shard) + X1, packed on the device (one sync)
  if (c.spmd) {
    CK(c.ft_cols.ensure((uint64_t)FCOLS * c.n_ftiles * 4)); CK(c.ft_base.ensure((uint64_t)FCOLS * c.n_ftiles * 4));
    CK(c.st_tot.ensure((uint64_t)c.PP * FCOLS * 4));
    CK(c.ft_posA.ensure((uint64_t)c.n_ftiles * c.FT * 4)); CK(c.ft_posB.ensure((uint64_t)c.n_ftiles * c.FT * 4));
    CK(c.ft_posK.ensure((uint64_t)c.n_ftiles * c.FT * 2));
    c.launches += timed(c, "k_fused_prepass", [&] { return launch_fused_prepass(c); });
    c.launches += timed(c, "k_fused_census", [&] { return launch_fused_census(c); });
  }
  const uint64_t nbm = c.n_bm_words;
  const size_t HA = 16, LA = HA + 2 * (size_t)nc + nbm;
  std::vector<uint32_t> AA;
  CK(c.x_send.ensure(LA * 4));
  k_x1_pack<<<(unsigned)std::min<uint64_t>((LA + 255) / 256, 1024), 256, 0, c.stream>>>(
      c.counters.as<Counters>(), c.spmd ? 0u : 1u, (unsigned long long)c.N, c.ch_nmin.as<uint32_t>(), c.ch_nmax.as<uint32_t>(),
      c.bitmap.as<uint32_t>(), nc, nbm, c.x_send.as<uint32_t>());
  c.launches += 1;
  timed(c, "x1_allgather", [&] { st = allgather_dev(c, LA, AA); return 0; });
  if (st) return st;
  auto hdr = [&](uint32_t s, size_t i) { return AA[(size_t)s * LA + i]; };
  auto u64at = [&](uint32_t s, size_t i) { return (uint64_t)hdr(s, i) | ((uint64_t)hdr(s, i + 1) << 32); };
  for (uint32_t s = 0; s < G; ++s) {  // identical data on every shard -> identical decisions
    const uint32_t x = hdr(s, 0);
    if (!x) continue;
    std::ostringstream m;
    if (x == 1) { m << "sharded analysis needs an SPMD trace on every shard (shard " << s << " is not)"; c.err = m.str(); return SCAN_E_UNSUPPORTED; }
    if (x == 2) { m << "schema error at event " << u64at(s, 7) << " of shard " << s; c.err = m.str(); return SCAN_E_SCHEMA; }
    m << "capacity exceeded on shard " << s; c.err = m.str(); return SCAN_E_UNSUPPORTED;
  }
  for (uint32_t s = 0; s + 1 < G; ++s) {
    if (hdr(s, 2) != hdr(s, 1) || hdr(s, 3) != W) {
      std::ostringstream m;
      m << "shard " << s << " does not end on an iteration boundary of every rank";
      c.err = m.str(); return SCAN_E_UNSUPPORTED;
    }
    for (uint32_t k = 0; k < nc; ++k)
      if (c.h_coff[k + 1] > c.h_coff[k] && hdr(s, HA + k) != hdr(s, HA + nc + k)) {
        std::ostringstream m;
        m << "communicator " << k << " has unequal member counts inside shard " << s;
        c.err = m.str(); return SCAN_E_UNSUPPORTED;
      }
  }
  uint32_t it_off = 0, n_iters = 0;
  for (uint32_t s = 0; s < G; ++s) {
    if (s < g) it_off += hdr(s, 1);
    n_iters += s + 1 < G ? hdr(s, 1) : hdr(s, 4);
  }
  c.it_off = it_off;
  {  // fresh host counters: census values from this shard's own header
    Counters z{};
    z.bad_event = ~0ull; z.min_niter = hdr(g, 2);
    z.max_niter = hdr(g, 1); z.n_end_ranks = hdr(g, 3); z.n_iters = hdr(g, 4);
    z.n_comm = u64at(g, 9); z.n_comp = u64at(g, 11); z.max_ncomp = hdr(g, 13); z.n_bits_words = u64at(g, 14);
    c.hc = z;
  }
  c.g_N = c.g_ncomm = c.g_ncomp = 0;
  for (uint32_t s = 0; s < G; ++s) { c.g_N += u64at(s, 5); c.g_ncomm += u64at(s, 9); c.g_ncomp += u64at(s, 11); }
  std::vector<uint32_t> bm(nbm, 0);  // job-wide P2P channel bitmap (OR over shards)
  uint64_t np = 0;
  for (uint32_t s = 0; s < G; ++s)
    for (uint64_t i = 0; i < nbm; ++i) bm[i] |= AA[(size_t)s * LA + HA + 2 * nc + i];
  for (uint64_t i = 0; i < nbm; ++i) np += (uint64_t)__builtin_popcount(bm[i]);
  if (nbm) CK(cudaMemcpyAsync(c.bitmap.p, bm.data(), nbm * 4, cudaMemcpyHostToDevice, c.stream));
  c.launches += timed(c, "k_rank_prefix", [&] { return launch_rank_prefix(c); });
  // ---- X2: P2P member counts per job-wide P2P channel
  const uint64_t NCH = nc + np;
  c.n_p2p = np; c.NCH = NCH; c.hc.n_p2p = np;
  CK(c.ch_nsend.ensure(std::max<uint64_t>(2 * np, 1) * 4)); CK(c.ch_nrecv.ensure(std::max<uint64_t>(2 * np, 1) * 4));
  if (np) {
    CK(cudaMemsetAsync(c.ch_nsend.p, 0, 2 * np * 4, c.stream));
    CK(cudaMemsetAsync(c.ch_nrecv.p, 0, 2 * np * 4, c.stream));
  }
  c.launches += timed(c, "k_p2p_counts", [&] { return launch_p2p_counts(c); });
  const size_t LB = std::max<size_t>(2 * np, 1);
  std::vector<uint32_t> BB;
  CK(c.x_send.ensure(LB * 4));
  CK(cudaMemsetAsync(c.x_send.p, 0, LB * 4, c.stream));
  if (np) {
    CK(cudaMemcpyAsync(c.x_send.p, c.ch_nsend.p, np * 4, cudaMemcpyDeviceToDevice, c.stream));
    CK(cudaMemcpyAsync(c.x_send.as<uint32_t>() + np, c.ch_nrecv.p, np * 4, cudaMemcpyDeviceToDevice, c.stream));
  }
  timed(c, "x2_allgather", [&] { st = allgather_dev(c, LB, BB); return 0; });
  if (st) return st;
  // P2P endpoints in channel order (ascending src*W + dst, the bitmap order)
  std::vector<uint32_t> psrc(np), pdst(np);
  {
    uint64_t p = 0;
    for (uint64_t wd = 0; wd < nbm; ++wd)
      for (uint32_t x = bm[wd]; x; x &= x - 1) {
        const uint64_t pair = wd * 32 + (uint64_t)__builtin_ctz(x);
        psrc[p] = (uint32_t)(pair / W); pdst[p] = (uint32_t)(pair % W); ++p;
      }
  }
  {  // job-wide P2P neighbour lists: they index the wait-for edge columns every shard sums into
    std::vector<std::vector<uint32_t>> peers(W);
    for (uint64_t p = 0; p < np; ++p) { peers[psrc[p]].push_back(pdst[p]); peers[pdst[p]].push_back(psrc[p]); }
    std::vector<uint32_t> nbp(W * PCAP, 0), nbpn(W, 0);
    for (uint64_t r = 0; r < W; ++r) {
      auto& v = peers[r];
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
      if (v.size() > (size_t)PCAP) { c.err = "capacity exceeded: more than 32 P2P peers on a rank"; return SCAN_E_UNSUPPORTED; }
      nbpn[r] = (uint32_t)v.size();
      for (size_t i = 0; i < v.size(); ++i) nbp[r * PCAP + i] = v[i];
    }
    CK(cudaMemcpyAsync(c.nbp.p, nbp.data(), W * PCAP * 4, cudaMemcpyHostToDevice, c.stream));
    CK(cudaMemcpyAsync(c.nbp_n.p, nbpn.data(), W * 4, cudaMemcpyHostToDevice, c.stream));
  }
  for (uint32_t s = 0; s + 1 < G; ++s)
    for (uint64_t p = 0; p < np; ++p)
      if (BB[(size_t)s * LB + p] != BB[(size_t)s * LB + np + p]) {
        std::ostringstream m;
        m << "P2P pair " << psrc[p] << "->" << pdst[p] << " has unequal send / recv counts inside shard " << s;
        c.err = m.str(); return SCAN_E_UNSUPPORTED;
      }
  // ---- job-wide channel tables (the unsharded k_channels numbering) + this shard's offsets
  auto nmem = [&](uint64_t ch) -> uint64_t { return ch < nc ? c.h_coff[ch + 1] - c.h_coff[ch] : 2; };
  auto lmax = [&](uint32_t s, uint64_t ch) -> uint32_t {
    if (ch < nc) return nmem(ch) ? AA[(size_t)s * LA + HA + nc + ch] : 0u;
    const uint64_t p = ch - nc;
    return std::max(BB[(size_t)s * LB + p], BB[(size_t)s * LB + np + p]);
  };
  auto lmin = [&](uint32_t s, uint64_t ch) -> uint32_t {
    if (ch < nc) return nmem(ch) ? AA[(size_t)s * LA + HA + ch] : 0u;
    const uint64_t p = ch - nc;
    return std::min(BB[(size_t)s * LB + p], BB[(size_t)s * LB + np + p]);
  };
  std::vector<uint64_t> gbase(NCH + 1), gslot(NCH + 1), kbase(NCH + 1), kslot(NCH + 1), pre(NCH), xb(NCH + 1);
  std::vector<uint32_t> gmax(NCH), gmin(NCH), lmx(NCH), lmn(NCH);
  uint64_t cb = 0, cs = 0, cx = 0;
  for (uint64_t ch = 0; ch < NCH; ++ch) {
    uint64_t tot = 0, pr = 0;
    for (uint32_t s = 0; s < G; ++s) { if (s == g) pr = tot; tot += lmax(s, ch); }
    gmax[ch] = (uint32_t)tot;
    gmin[ch] = (uint32_t)(tot - lmax(G - 1, ch) + lmin(G - 1, ch));
    lmx[ch] = lmax(g, ch); lmn[ch] = lmin(g, ch);
    gbase[ch] = cb; gslot[ch] = cs; pre[ch] = pr;
    kbase[ch] = cb + pr; kslot[ch] = cs + pr * nmem(ch);
    xb[ch] = cx;
    if (ch >= nc || (c.h_ccls[ch] != 1 && c.h_ccls[ch] != 2)) cx += lmx[ch];
    cb += tot; cs += tot * nmem(ch);
  }
  gbase[NCH] = kbase[NCH] = cb; gslot[NCH] = kslot[NCH] = cs; xb[NCH] = cx;
  if (cb >= 0xFFFFFFFFull) { c.err = "more than 2^32-1 instances"; return SCAN_E_UNSUPPORTED; }
  if (n_iters >= (1u << 24)) { c.err = "sharded analysis supports < 2^24 iterations"; return SCAN_E_UNSUPPORTED; }
  CK(c.ch_base.ensure((NCH + 1) * 8)); CK(c.ch_slot.ensure((NCH + 1) * 8)); CK(c.xbase.ensure((NCH + 1) * 8));
  if ((st = upload(c, c.ch_base, kbase)) || (st = upload(c, c.ch_slot, kslot)) || (st = upload(c, c.xbase, xb)) ||
      (st = upload(c, c.g_base, gbase)) || (st = upload(c, c.g_slot, gslot)) || (st = upload(c, c.g_nmax, gmax)) ||
      (st = upload(c, c.g_nmin, gmin)) || (st = upload(c, c.g_k0, pre)))
    return st;
  CK(cudaMemcpyAsync(c.ch_nmax.p, lmx.data(), NCH * 4, cudaMemcpyHostToDevice, c.stream));
  CK(cudaMemcpyAsync(c.ch_nmin.p, lmn.data(), NCH * 4, cudaMemcpyHostToDevice, c.stream));
  if (np) {
    CK(cudaMemcpyAsync(c.ch_nsend.as<uint32_t>() + np, psrc.data(), np * 4, cudaMemcpyHostToDevice, c.stream));
    CK(cudaMemcpyAsync(c.ch_nrecv.as<uint32_t>() + np, pdst.data(), np * 4, cudaMemcpyHostToDevice, c.stream));
  }
  c.h_shard_k0 = pre; c.h_shard_n = lmx;
  c.hc.n_instances = cb; c.hc.n_slots = cs; c.hc.p2p_inst0 = gbase[nc]; c.hc.p2p_slot0 = gslot[nc];
  c.hc.n_xinst = cx; c.hc.n_iters = n_iters;
  c.n_comm = c.hc.n_comm; c.n_comp = c.hc.n_comp; c.NIT = c.hc.max_niter; c.n_iters = n_iters;
  c.max_ncomp = c.hc.max_ncomp; c.n_bits_words = c.hc.n_bits_words;
  c.n_inst = cb; c.n_slots = cs; c.p2p_slot0 = gslot[nc]; c.p2p_inst0 = gbase[nc]; c.n_xinst = cx;
  CK(cudaMemcpyAsync(c.counters.p, &c.hc, sizeof(Counters), cudaMemcpyHostToDevice, c.stream));
  if ((st = alloc_match_buffers(c, true))) return st;
  // ---- local fused pass (K9 + cross-stage reduce + deferred stage 2), job-wide ids / windows
  if ((st = alloc_detect(c)) || (st = alloc_localize(c))) return st;
  CK(c.dlate.ensure((uint64_t)c.n_ftiles * ((c.FR + 31) / 32) * 4 + 4));
  CK(cudaMemsetAsync(c.dlate.p, 0, (uint64_t)c.n_ftiles * ((c.FR + 31) / 32) * 4 + 4, c.stream));
  CK(c.dinfo.ensure((uint64_t)c.n_ftiles * 16 + 16));
  const uint64_t items = (uint64_t)c.NW * W, nlk = (uint64_t)c.NW * np, ncl = (uint64_t)c.TP * c.PP;
  CK(cudaMemsetAsync(c.wd_total.p, 0, items * 4, c.stream));
  CK(cudaMemsetAsync(c.wd_slow.p, 0, items * 4, c.stream));
  c.launches += timed(c, "k_class_counts", [&] { return launch_class_counts(c); });
  c.launches += timed(c, "k_fused", [&] { return launch_fused(c); });
  c.launches += timed(c, "k_cross_reduce", [&] { return launch_cross_reduce(c); });
  c.launches += timed(c, "k_deferred", [&] { return launch_deferred(c); });
  // ---- X3: P2P instance records to the owner of their link (pid % G)
  std::vector<LinkMap> smap, rmap;
  std::vector<size_t> scount(G, 0), rcount(G, 0), soff(G + 1, 0), roff(G + 1, 0);
  {
    uint64_t flat = 0;
    for (uint32_t d = 0; d < G; ++d) {
      soff[d] = flat;
      if (d != g)
        for (uint64_t p = d; p < np; p += G) {
          const uint64_t ch = nc + p;
          const uint32_t n = lmx[ch];
          if (n) { smap.push_back({flat, kbase[ch], kslot[ch], n, 0}); flat += n; }
        }
      scount[d] = flat - soff[d];
    }
    soff[G] = flat;
    flat = 0;
    for (uint32_t s = 0; s < G; ++s) {
      roff[s] = flat;
      if (s != g)
        for (uint64_t p = g; p < np; p += G) {
          const uint64_t ch = nc + p;
          const uint32_t n = lmax(s, ch);
          uint64_t pr = 0;
          for (uint32_t q = 0; q < s; ++q) pr += lmax(q, ch);
          if (n) { rmap.push_back({flat, gbase[ch] + pr, gslot[ch] + 2 * pr, n, 0}); flat += n; }
        }
      rcount[s] = flat - roff[s];
    }
    roff[G] = flat;
  }
  if (G > 1 && np) {
    if ((st = upload(c, c.lk_sendmap, smap)) || (st = upload(c, c.lk_recvmap, rmap))) return st;
    CK(c.x_send.ensure(std::max<size_t>(soff[G], 1) * LREC * 4));
    CK(c.x_recv.ensure(std::max<size_t>(roff[G], 1) * LREC * 4));
    if (!smap.empty()) {
      k_link_pack<<<(unsigned)smap.size(), 256, 0, c.stream>>>(c.lk_sendmap.as<LinkMap>(), c.inst_rec.as<uint4>(),
                                                              c.p2p_iter.as<uint32_t>(), c.p2p_pay.as<uint32_t>(),
                                                              c.p2p_inst0, c.p2p_slot0, c.x_send.as<uint32_t>());
      c.launches += 1;
    }
    ncclResult_t xr = ncclSuccess;
    timed(c, "x3_alltoall", [&] {
      ncclGroupStart();
      for (uint32_t d = 0; d < G; ++d) {
        if (d == g) continue;
        if (scount[d]) ncclSend(c.x_send.as<uint32_t>() + soff[d] * LREC, scount[d] * LREC, ncclUint32, (int)d, comm, c.stream);
        if (rcount[d]) ncclRecv(c.x_recv.as<uint32_t>() + roff[d] * LREC, rcount[d] * LREC, ncclUint32, (int)d, comm, c.stream);
      }
      xr = ncclGroupEnd();
      return 0;
    });
    if (xr != ncclSuccess) { c.err = std::string("NCCL all-to-all: ") + ncclGetErrorString(xr); return SCAN_E_NCCL; }
    if (!rmap.empty()) {
      k_link_unpack<<<(unsigned)rmap.size(), 256, 0, c.stream>>>(c.lk_recvmap.as<LinkMap>(), c.x_recv.as<uint32_t>(),
                                                                c.inst_rec.as<uint4>(), c.p2p_iter.as<uint32_t>(),
                                                                c.p2p_pay.as<uint32_t>(), c.p2p_inst0, c.p2p_slot0);
      c.launches += 1;
    }
  }
  c.launches += timed(c, "k_link_median", [&] { return launch_link_median(c); });
  // ---- stage-2 boundary records of this shard's ranks
  CK(c.headtail.ensure(((uint64_t)G * W + 16) * 8));
  CK(cudaMemsetAsync(c.headtail.p, 0, ((uint64_t)G * W + 16) * 8, c.stream));
  unsigned long long* ht = c.headtail.as<unsigned long long>();
  c.launches += timed(c, "k_shard_head", [&] {
    k_shard_head<<<(unsigned)((W + 7) / 8), 256, 0, c.stream>>>(
        c.W, c.rank_off.as<uint64_t>(), c.d_kind, c.r_comm_off.as<uint64_t>(), c.r_bits_off.as<uint64_t>(),
        c.r_ncomp.as<uint32_t>(), c.bits.as<uint32_t>(), c.inst_c.as<uint32_t>(), c.inst_rec.as<uint4>(),
        c.lcfg.stage2_classes, (unsigned long long)c.lcfg.late_margin_ns, c.dcfg.window_iters, c.it_off, ht + (uint64_t)g * W);
    return 1;
  });
  // this shard's status + match counters ride along in the last 16 words of the record buffer
  {
    k_x4_status<<<1, 32, 0, c.stream>>>(c.counters.as<Counters>(), c.cl_J.as<uint32_t>(), c.cl_max.as<uint32_t>(),
                                        (uint32_t)ncl, (g + 1 < G && c.DP >= 2) ? 1 : 0, ht + (uint64_t)G * W);
    c.launches += 1;
    unsigned long long e[16];
    // ---- X4: one grouped all-reduce (sum) of every partial result
    const uint64_t nnz_tot = c.nnz_c + W * PCAP;
    ncclResult_t xr = ncclSuccess;
    timed(c, "x4_allreduce", [&] {
      ncclGroupStart();
      auto ar = [&](DevBuf& b, uint64_t n, ncclDataType_t t) { if (n) ncclAllReduce(b.p, b.p, n, t, ncclSum, comm, c.stream); };
      ar(c.wd_total, items, ncclUint32); ar(c.wd_slow, items, ncclUint32);
      ar(c.wl_joined, items, ncclUint32); ar(c.wl_late, items, ncclUint32);
      ar(c.lk_n, nlk, ncclUint32); ar(c.lk_medp, nlk, ncclUint32); ar(c.lk_medt, nlk, ncclUint32);
      ar(c.lk_used, nlk, ncclUint8); ar(c.lk_elig, nlk, ncclUint8); ar(c.lk_bw, nlk, ncclFloat64);
      ar(c.cl_J, ncl, ncclUint32); ar(c.cl_max, ncl, ncclUint32);
      ar(c.ewc, (uint64_t)c.NW * nnz_tot, ncclUint64); ar(c.rk_sum, 3 * W, ncclUint64);
      ar(c.headtail, (uint64_t)G * W + 16, ncclUint64);
      xr = ncclGroupEnd();
      return 0;
    });
    if (xr != ncclSuccess) { c.err = std::string("NCCL all-reduce: ") + ncclGetErrorString(xr); return SCAN_E_NCCL; }
    CK(cudaMemcpyAsync(e, ht + (uint64_t)G * W, sizeof(e), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    if (e[0]) { c.err = "sharded analysis needs an SPMD trace on every shard (fused-pass verification failed)"; return SCAN_E_UNSUPPORTED; }
    if (e[1]) { c.err = "a DP class has unequal compute counts inside a shard other than the last"; return SCAN_E_UNSUPPORTED; }
    c.hc.n_incomplete = e[2]; c.hc.n_kind_mismatch = e[3]; c.hc.n_payload_mismatch = e[4];
  }
  // ---- replicated tail on identical job-wide inputs
  {
    Counters z = c.hc;
    z.n_compared = z.n_slow = z.n_candidates = z.n_class_mismatch = 0;
    z.n_link_slow = z.n_roots = z.n_victims = z.n_unattributed = 0;
    for (auto& v : z.v_count) v = 0;
    CK(cudaMemcpyAsync(c.counters.p, &z, sizeof(Counters), cudaMemcpyHostToDevice, c.stream));
  }
  if (c.lcfg.stage2_mode == 0 && G > 1) {
    k_shard_fixup<<<(unsigned)((W + 255) / 256), 256, 0, c.stream>>>(c.W, (int)G, ht, c.wl_joined.as<uint32_t>(),
                                                                     c.wl_late.as<uint32_t>());
    c.launches += 1;
  }
  c.launches += timed(c, "k_wd_finish", [&] { return launch_wd_finish(c); });
  c.launches += timed(c, "k_link_flags", [&] { return launch_link_flags(c); });
  c.launches += timed(c, "k_walk", [&] { return launch_verdict_walk(c); });
  if ((st = sync_read(c))) return st;
  if (c.hc.overflow & 24u) {
    c.err = "capacity exceeded: more than 16384 samples on a link / links in a direction class";
    return SCAN_E_UNSUPPORTED;
  }
  c.matched = c.detected = c.localized = true;
  c.fused_used = true;
  c.xwait_pending = true;
  return SCAN_OK;
}

void shard_release(Ctx& c) {
  if (c.nccl) ncclCommDestroy((ncclComm_t)c.nccl);
  c.nccl = nullptr;
}

}  // namespace ms

using namespace ms;

extern "C" {

scan_status scan_nccl_unique_id(uint8_t out[128]) {
  if (!out) return SCAN_E_INVALID_ARG;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return SCAN_E_NCCL;
  std::memcpy(out, &id, sizeof(id));
  return SCAN_OK;
}

scan_status scan_create_sharded(scan_ctx** out, int cuda_device, void* cuda_stream, int n_shards, int shard,
                                const uint8_t nccl_unique_id[128]) {
  if (!out || n_shards < 1 || shard < 0 || shard >= n_shards || (n_shards > 1 && !nccl_unique_id)) return SCAN_E_INVALID_ARG;
  scan_status st = scan_create(out, cuda_device, cuda_stream);
  if (st) return st;
  Ctx& c = (*out)->c;
  c.n_shards = n_shards; c.shard = shard;
  if (n_shards > 1) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    ncclComm_t comm = nullptr;
    const ncclResult_t r = ncclCommInitRank(&comm, n_shards, id, shard);
    if (r != ncclSuccess) {
      c.err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
      return SCAN_E_NCCL;  // the context stays valid (caller destroys it); scan_last_error has the reason
    }
    c.nccl = comm;
  }
  return SCAN_OK;
}

}  // extern "C"
