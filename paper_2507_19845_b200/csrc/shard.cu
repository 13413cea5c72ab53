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
#include <chrono>
#include <cstdio>
#include <cstdlib>
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
// (a P2P instance i's send slot, SlotRec: p2p_slot0 + 2 (i - p2p_inst0), payload in w, iteration in z)
__global__ void k_link_pack(const LinkMap* map, const uint4* rec, const uint4* slots, uint64_t p2p_inst0, uint64_t p2p_slot0,
                            uint32_t* buf) {
  const LinkMap m = map[blockIdx.x];
  for (uint32_t k = threadIdx.x; k < m.n; k += blockDim.x) {
    const uint64_t i = m.inst0 + k;
    const uint4 r = rec[i];
    uint32_t* o = buf + (m.flat + k) * LREC;
    uint4 sl = make_uint4(0, 0, 0, 0);
    if (r.w & SCAN_F_COMPLETE) sl = slots[p2p_slot0 + 2 * (i - p2p_inst0)];  // both slots written: the window
                                                                              // search reads complete instances
    o[0] = r.x;
    o[1] = sl.w;
    o[2] = ((sl.z & SLOT_IT_MASK) << 8) | (r.w & 0xFFu);
  }
}

// rows of links this shard owns; only the fields the median reads are written (the rest of an
// unowned-range row stays unspecified, scan.h)
__global__ void k_link_unpack(const LinkMap* map, const uint32_t* buf, uint4* rec, uint4* slots, unsigned long long* lk_key,
                              uint64_t p2p_inst0, uint64_t p2p_slot0) {
  const LinkMap m = map[blockIdx.x];
  for (uint32_t k = threadIdx.x; k < m.n; k += blockDim.x) {
    const uint64_t i = m.inst0 + k;
    const uint32_t* v = buf + (m.flat + k) * LREC;
    rec[i].x = v[0];
    rec[i].w = v[2] & 0xFFu;
    uint32_t* sw = reinterpret_cast<uint32_t*>(slots + p2p_slot0 + 2 * (i - p2p_inst0));
    sw[2] = v[2] >> 8;  // iteration (the warm-up flag travels in the record's flags)
    sw[3] = v[1];
    lk_key[i - p2p_inst0] = lk_sample_key(v[2] & 0xFFu, v[0], v[1]);
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

// OR of every shard's P2P channel bitmap (rows of the gathered X1 buffer)
__global__ void k_bitmap_or(const uint32_t* gathered, uint64_t stride, uint64_t off, uint64_t nbm, uint32_t G, uint32_t* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nbm; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    for (uint32_t s = 0; s < G; ++s) v |= gathered[s * stride + off + i];
    out[i] = v;
  }
}

// (src, dst) of every job-wide P2P channel (channel id = popcount prefix, ascending src*W + dst)
__global__ void k_p2p_endpoints(uint32_t W, const uint32_t* bitmap, const uint32_t* bitpre, uint64_t nbm, uint32_t* psrc,
                                uint32_t* pdst) {
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nbm; w += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t x = bitmap[w], id = bitpre[w];
    while (x) {
      const uint64_t pair = w * 32 + (uint64_t)(__ffs(x) - 1);
      psrc[id] = (uint32_t)(pair / W); pdst[id] = (uint32_t)(pair % W);
      ++id; x &= x - 1;
    }
  }
}

// job-wide P2P neighbour list of every rank (ascending; they index the wait-for edge columns all
// shards sum into): d is a neighbour of r iff a channel r->d or d->r exists. One warp per rank,
// lanes over candidate neighbours, ballot compaction keeps the order.
__global__ void k_p2p_peers(uint32_t W, const uint32_t* bitmap, uint32_t* nbp, uint32_t* nbp_n, Counters* cnt) {
  const uint32_t r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= W) return;
  const uint32_t lane = lane_id();
  uint32_t n = 0;
  bool over = false;
  for (uint32_t d0 = 0; d0 < W; d0 += 32) {
    const uint32_t d = d0 + lane;
    bool e = false;
    if (d < W && d != r) {
      const uint64_t x = (uint64_t)r * W + d, y = (uint64_t)d * W + r;
      e = ((bitmap[x >> 5] >> (x & 31)) & 1u) | ((bitmap[y >> 5] >> (y & 31)) & 1u);
    }
    const unsigned m = __ballot_sync(0xFFFFFFFFu, e);
    const uint32_t pos = n + __popc(m & ((1u << lane) - 1u));
    if (e && pos < (uint32_t)PCAP) nbp[(uint64_t)r * PCAP + pos] = d;
    n += __popc(m);
    if (n > (uint32_t)PCAP) { over = true; break; }
  }
  if (lane == 0) {
    nbp_n[r] = over ? (uint32_t)PCAP : n;
    if (over) atomicOr(&cnt->overflow, 4u);
  }
}

// scatter of the staged host tables into their device buffers (one launch instead of a copy each)
struct Unstage { const uint8_t* src; uint8_t* dst[12]; uint64_t off[12], bytes[12]; int n; };
__global__ void k_unstage(Unstage u) {
  for (int k = 0; k < u.n; ++k)
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < u.bytes[k]; i += (uint64_t)gridDim.x * blockDim.x)
      u.dst[k][i] = u.src[u.off[k] + i];
}

// X2 send row: this shard's send / recv counts of the n_p2p job-wide channels, zero-padded to cap
__global__ void k_x2_pack(const Counters* cnt, const uint32_t* nsend, const uint32_t* nrecv, uint64_t cap, uint32_t* out) {
  const uint64_t np = cnt->n_p2p;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 2 * cap; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = i < np ? nsend[i] : (i < 2 * np ? nrecv[i - np] : 0u);
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

// after X4: the job-wide integrity counters into the replicated tail's counters (no host round trip)
__global__ void k_x4_apply(const unsigned long long* e, Counters* cnt) {
  if (threadIdx.x || blockIdx.x) return;
  cnt->n_incomplete = e[2]; cnt->n_kind_mismatch = e[3]; cnt->n_payload_mismatch = e[4];
}

// pinned host scratch of the shard path (exchange read-backs, table staging)
scan_status pin_ensure(Ctx& c, size_t bytes) {
  if (bytes <= c.h_pin_cap && c.h_pin) return SCAN_OK;
  if (c.h_pin) { CK(cudaStreamSynchronize(c.stream)); cudaFreeHost(c.h_pin); c.h_pin = nullptr; c.h_pin_cap = 0; }
  CK(cudaMallocHost(&c.h_pin, bytes));
  c.h_pin_cap = bytes;
  return SCAN_OK;
}
// grow, keeping the current contents (read-backs already landed: the stream is synchronised)
scan_status pin_ensure_keep(Ctx& c, size_t bytes) {
  if (bytes <= c.h_pin_cap && c.h_pin) return SCAN_OK;
  void* nb = nullptr;
  CK(cudaMallocHost(&nb, bytes));
  if (c.h_pin) { std::memcpy(nb, c.h_pin, c.h_pin_cap); cudaFreeHost(c.h_pin); }
  c.h_pin = nb; c.h_pin_cap = bytes;
  return SCAN_OK;
}

}  // namespace

scan_status sharded_all(Ctx& c) {
  // MS_SHARD_PROFILE=1: host-side phase timestamps on stderr (diagnostics)
  static const bool prof = std::getenv("MS_SHARD_PROFILE") != nullptr;
  using clk = std::chrono::steady_clock;
  const auto t_start = clk::now();
  std::vector<std::pair<const char*, double>> marks;
  auto mark = [&](const char* what) {
    if (prof) marks.push_back({what, std::chrono::duration<double, std::micro>(clk::now() - t_start).count()});
  };
  struct Dump {
    std::vector<std::pair<const char*, double>>& m; int g;
    ~Dump() {
      if (m.empty()) return;
      std::fprintf(stderr, "[shard %d]", g);
      for (auto& x : m) std::fprintf(stderr, " %s=%.0f", x.first, x.second);
      std::fprintf(stderr, " (us)\n");
    }
  } dump{marks, c.shard};
  c.matched = c.detected = c.localized = false;
  c.fused_used = false; c.tiles_ready = false; c.xwait_pending = false;
  const uint32_t G = (uint32_t)c.n_shards, g = (uint32_t)c.shard, nc = c.n_comms;
  const uint64_t W = c.W;
  scan_status st;
  if ((st = prep_ws(c, false))) return st;
  // ---- local census (the fused pre-pass of this shard) + X1, packed on the device (one sync)
  if (c.spmd) {
    CK(c.ft_cols.ensure((uint64_t)FCOLS * c.n_ftiles * 4)); CK(c.ft_base.ensure((uint64_t)FCOLS * c.n_ftiles * 4));
    CK(c.st_tot.ensure((uint64_t)c.PP * FCOLS * 4));
    CK(c.ft_posA.ensure((uint64_t)c.n_ftiles * c.FT * 4)); CK(c.ft_posB.ensure((uint64_t)c.n_ftiles * c.FT * 4));
    if (c.use_stage) CK(c.ft_tbase.ensure((uint64_t)c.n_ftiles * 40 * 4));
    CK(c.ft_posK.ensure((uint64_t)c.n_ftiles * c.FT * 2));
    c.launches += timed(c, "k_fused_prepass", [&] { return launch_fused_prepass(c); });
    c.launches += timed(c, "k_fused_census", [&] { return launch_fused_census(c); });
  }
  const uint64_t nbm = c.n_bm_words;
  const size_t HA = 16, HL = HA + 2 * (size_t)nc, LA = HL + nbm;  // X1 row: header | nmin | nmax | bitmap
  const uint64_t NPMAX = W * PCAP;                                  // P2P channels <= ranks x peers
  const size_t LB = 2 * NPMAX;                                      // X2 row: nsend | nrecv (fixed capacity)
  // pinned host regions: A = X1 rows without bitmaps, C = counters, B = X2 rows (2*np used), D = staging
  const size_t offA = 0, offC = (offA + (size_t)G * HL * 4 + 63) & ~size_t(63), offB = (offC + sizeof(Counters) + 63) & ~size_t(63);
  CK(c.x_send.ensure(std::max(LA, LB) * 4)); CK(c.x_recv.ensure((size_t)G * LA * 4)); CK(c.x_recv2.ensure((size_t)G * LB * 4));
  CK(c.ch_nsend.ensure(LB * 4)); CK(c.ch_nrecv.ensure(LB * 4)); CK(c.x_ep.ensure(LB * 4));
  CK(cudaMemsetAsync(c.ch_nsend.p, 0, NPMAX * 4, c.stream));
  CK(cudaMemsetAsync(c.ch_nrecv.p, 0, NPMAX * 4, c.stream));
  if (!c.ev_x1) { CK(cudaEventCreateWithFlags(&c.ev_x1, cudaEventDisableTiming)); CK(cudaEventCreateWithFlags(&c.ev_x2, cudaEventDisableTiming)); }
  if ((st = pin_ensure(c, offB + (size_t)G * LB * 4))) return st;
  uint8_t* pin = static_cast<uint8_t*>(c.h_pin);
  // ---- X1 (device-packed) and, right behind it, the device-side P2P channel set and X2: no host
  // round trip between the two all-gathers
  flush_fills(c);  // prep_ws fills (channel count extremes, bitmap) precede the census
  k_x1_pack<<<(unsigned)std::min<uint64_t>((LA + 255) / 256, 1024), 256, 0, c.stream>>>(
      c.counters.as<Counters>(), c.spmd ? 0u : 1u, (unsigned long long)c.N, c.ch_nmin.as<uint32_t>(), c.ch_nmax.as<uint32_t>(),
      c.bitmap.as<uint32_t>(), nc, nbm, c.x_send.as<uint32_t>());
  c.launches += 1;
  mark("launch");
  int xr = 0;
  timed(c, "x1_allgather", [&] { xr = xch_allgather(c, c.x_send.p, c.x_recv.p, LA); return 0; });
  if (xr) { c.err = std::string("exchange all-gather: ") + xch_error(xr); return SCAN_E_NCCL; }
  CK(cudaMemcpy2DAsync(pin + offA, HL * 4, c.x_recv.p, LA * 4, HL * 4, G, cudaMemcpyDeviceToHost, c.stream));
  CK(cudaEventRecord(c.ev_x1, c.stream));
  // the device-side P2P channel set needs this shard's census: a shard that is not SPMD skips it (its X1
  // header makes every shard return UNSUPPORTED right after X2; the X2 words it sends are zeros)
  if (c.spmd) c.launches += timed(c, "k_p2p_set", [&] {
    k_bitmap_or<<<(unsigned)std::min<uint64_t>((nbm + 255) / 256, 4096), 256, 0, c.stream>>>(
        c.x_recv.as<uint32_t>(), LA, HL, nbm, G, c.bitmap.as<uint32_t>());
    launch_rank_prefix(c);  // channel ids = popcount prefix of the job-wide bitmap; n_p2p
    k_p2p_endpoints<<<(unsigned)std::min<uint64_t>((nbm + 255) / 256, 4096), 256, 0, c.stream>>>(
        (uint32_t)W, c.bitmap.as<uint32_t>(), c.bitpre.as<uint32_t>(), nbm, c.x_ep.as<uint32_t>(), c.x_ep.as<uint32_t>() + NPMAX);
    k_p2p_peers<<<(unsigned)((W + 7) / 8), 256, 0, c.stream>>>((uint32_t)W, c.bitmap.as<uint32_t>(), c.nbp.as<uint32_t>(),
                                                              c.nbp_n.as<uint32_t>(), c.counters.as<Counters>());
    launch_p2p_counts_to(c, c.ch_nsend.as<uint32_t>(), c.ch_nrecv.as<uint32_t>(), c.x_ep.as<uint32_t>(),
                         c.x_ep.as<uint32_t>() + NPMAX);
    return 5;
  });
  k_x2_pack<<<(unsigned)std::min<uint64_t>((LB + 255) / 256, 4096), 256, 0, c.stream>>>(
      c.counters.as<Counters>(), c.ch_nsend.as<uint32_t>(), c.ch_nrecv.as<uint32_t>(), NPMAX, c.x_send.as<uint32_t>());
  c.launches += 1;
  CK(cudaMemcpyAsync(pin + offC, c.counters.p, sizeof(Counters), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaEventRecord(c.ev_x2, c.stream));
  timed(c, "x2_allgather", [&] { xr = xch_allgather(c, c.x_send.p, c.x_recv2.p, LB); return 0; });
  if (xr) { c.err = std::string("exchange all-gather: ") + xch_error(xr); return SCAN_E_NCCL; }
  // host: X1 headers while the device works on the P2P channel set (identical data on every shard ->
  // identical decisions; every shard has enqueued the same collectives before any early return)
  CK(cudaEventSynchronize(c.ev_x1));
  mark("x1");
  const uint32_t* AA = reinterpret_cast<const uint32_t*>(pin + offA);
  auto hdr = [&](uint32_t s, size_t i) { return AA[(size_t)s * HL + i]; };
  auto u64at = [&](uint32_t s, size_t i) { return (uint64_t)hdr(s, i) | ((uint64_t)hdr(s, i + 1) << 32); };
  auto fail_all = [&](scan_status code, const std::string& m) { CK(cudaStreamSynchronize(c.stream)); c.err = m; return code; };
  for (uint32_t s = 0; s < G; ++s) {
    const uint32_t x = hdr(s, 0);
    if (!x) continue;
    std::ostringstream m;
    if (x == 1) { m << "sharded analysis needs an SPMD trace on every shard (shard " << s << " is not)"; return fail_all(SCAN_E_UNSUPPORTED, m.str()); }
    if (x == 2) { m << "schema error at event " << u64at(s, 7) << " of shard " << s; return fail_all(SCAN_E_SCHEMA, m.str()); }
    m << "capacity exceeded on shard " << s;
    return fail_all(SCAN_E_UNSUPPORTED, m.str());
  }
  for (uint32_t s = 0; s + 1 < G; ++s) {
    if (hdr(s, 2) != hdr(s, 1) || hdr(s, 3) != W) {
      std::ostringstream m;
      m << "shard " << s << " does not end on an iteration boundary of every rank";
      return fail_all(SCAN_E_UNSUPPORTED, m.str());
    }
    for (uint32_t k = 0; k < nc; ++k)
      if (c.h_coff[k + 1] > c.h_coff[k] && hdr(s, HA + k) != hdr(s, HA + nc + k)) {
        std::ostringstream m;
        m << "communicator " << k << " has unequal member counts inside shard " << s;
        return fail_all(SCAN_E_UNSUPPORTED, m.str());
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
  // P2P channel count (device prefix of the OR'ed bitmap), then exactly the X2 words in use
  CK(cudaEventSynchronize(c.ev_x2));
  const Counters* dc = reinterpret_cast<const Counters*>(pin + offC);
  const uint64_t np = dc->n_p2p;
  if (dc->overflow & 4u) return fail_all(SCAN_E_UNSUPPORTED, "capacity exceeded: more than 32 P2P peers on a rank");
  const size_t LBu = std::max<size_t>(2 * np, 1);
  if (np) CK(cudaMemcpy2DAsync(pin + offB, LBu * 4, c.x_recv2.p, LB * 4, 2 * np * 4, G, cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  mark("x2");
  const uint32_t* BB = reinterpret_cast<const uint32_t*>(pin + offB);
  const uint64_t NCH = nc + np;
  c.n_p2p = np; c.NCH = NCH; c.hc.n_p2p = np;
  for (uint32_t s = 0; s + 1 < G; ++s)
    for (uint64_t p = 0; p < np; ++p)
      if (BB[(size_t)s * LBu + p] != BB[(size_t)s * LBu + np + p]) {
        std::ostringstream m;
        m << "P2P channel " << p << " has unequal send / recv counts inside shard " << s;
        c.err = m.str(); return SCAN_E_UNSUPPORTED;
      }
  // ---- job-wide channel tables (the unsharded k_channels numbering) + this shard's offsets
  auto nmem = [&](uint64_t ch) -> uint64_t { return ch < nc ? c.h_coff[ch + 1] - c.h_coff[ch] : 2; };
  auto lmax = [&](uint32_t s, uint64_t ch) -> uint32_t {
    if (ch < nc) return nmem(ch) ? hdr(s, HA + nc + ch) : 0u;
    const uint64_t p = ch - nc;
    return std::max(BB[(size_t)s * LBu + p], BB[(size_t)s * LBu + np + p]);
  };
  auto lmin = [&](uint32_t s, uint64_t ch) -> uint32_t {
    if (ch < nc) return nmem(ch) ? hdr(s, HA + ch) : 0u;
    const uint64_t p = ch - nc;
    return std::min(BB[(size_t)s * LBu + p], BB[(size_t)s * LBu + np + p]);
  };
  // staging layout (u64 arrays, then u32 arrays) in pinned memory after region B; one H2D copy
  const size_t n1 = NCH + 1, offD = (offB + (size_t)G * LBu * 4 + 63) & ~size_t(63);
  const size_t bytesD = 5 * n1 * 8 + NCH * 8 + 4 * NCH * 4 + sizeof(Counters) + 64;
  if ((st = pin_ensure_keep(c, offD + bytesD))) return st;
  pin = static_cast<uint8_t*>(c.h_pin);
  BB = reinterpret_cast<const uint32_t*>(pin + offB);
  AA = reinterpret_cast<const uint32_t*>(pin + offA);
  uint64_t* gbase = reinterpret_cast<uint64_t*>(pin + offD);
  uint64_t* gslot = gbase + n1;
  uint64_t* kbase = gslot + n1;
  uint64_t* kslot = kbase + n1;
  uint64_t* xb = kslot + n1;
  uint64_t* pre = xb + n1;
  uint32_t* gmax = reinterpret_cast<uint32_t*>(pre + NCH);
  uint32_t* gmin = gmax + NCH;
  uint32_t* lmx = gmin + NCH;
  uint32_t* lmn = lmx + NCH;
  Counters* hcs = reinterpret_cast<Counters*>((reinterpret_cast<uintptr_t>(lmn + NCH) + 15) & ~uintptr_t(15));
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
  c.h_shard_k0.assign(pre, pre + NCH); c.h_shard_n.assign(lmx, lmx + NCH);
  c.hc.n_instances = cb; c.hc.n_slots = cs; c.hc.p2p_inst0 = gbase[nc]; c.hc.p2p_slot0 = gslot[nc];
  c.hc.n_xinst = cx; c.hc.n_iters = n_iters;
  c.n_comm = c.hc.n_comm; c.n_comp = c.hc.n_comp; c.NIT = c.hc.max_niter; c.n_iters = n_iters;
  c.max_ncomp = c.hc.max_ncomp; c.n_bits_words = c.hc.n_bits_words;
  c.n_inst = cb; c.n_slots = cs; c.p2p_slot0 = gslot[nc]; c.p2p_inst0 = gbase[nc]; c.n_xinst = cx;
  *hcs = c.hc;
  {  // one H2D of the staged tables, then device-side scatters into their buffers
    const size_t used = reinterpret_cast<uint8_t*>(hcs + 1) - (pin + offD);
    CK(c.x_stage.ensure(used));
    CK(cudaMemcpyAsync(c.x_stage.p, pin + offD, used, cudaMemcpyHostToDevice, c.stream));
    CK(c.ch_base.ensure(n1 * 8)); CK(c.ch_slot.ensure(n1 * 8)); CK(c.xbase.ensure(n1 * 8));
    CK(c.g_base.ensure(n1 * 8)); CK(c.g_slot.ensure(n1 * 8)); CK(c.g_k0.ensure(NCH * 8 + 8));
    CK(c.g_nmax.ensure(NCH * 4 + 4)); CK(c.g_nmin.ensure(NCH * 4 + 4));
    const cudaMemcpyKind dd = cudaMemcpyDeviceToDevice;
    Unstage u{static_cast<const uint8_t*>(c.x_stage.p), {}, {}, {}, 0};
    auto add = [&](DevBuf& d, const void* h, uint64_t bytes) {
      u.dst[u.n] = static_cast<uint8_t*>(d.p); u.off[u.n] = static_cast<const uint8_t*>(h) - (pin + offD); u.bytes[u.n] = bytes; ++u.n;
    };
    add(c.g_base, gbase, n1 * 8); add(c.g_slot, gslot, n1 * 8); add(c.ch_base, kbase, n1 * 8); add(c.ch_slot, kslot, n1 * 8);
    add(c.xbase, xb, n1 * 8); add(c.g_k0, pre, NCH * 8); add(c.g_nmax, gmax, NCH * 4); add(c.g_nmin, gmin, NCH * 4);
    add(c.ch_nmax, lmx, NCH * 4); add(c.ch_nmin, lmn, NCH * 4); add(c.counters, hcs, sizeof(Counters));
    k_unstage<<<64, 256, 0, c.stream>>>(u);
    c.launches += 1;
    if (np) {  // endpoints behind the counts (the layout every P2P consumer reads)
      CK(cudaMemcpyAsync(c.ch_nsend.as<uint32_t>() + np, c.x_ep.p, np * 4, dd, c.stream));
      CK(cudaMemcpyAsync(c.ch_nrecv.as<uint32_t>() + np, c.x_ep.as<uint32_t>() + NPMAX, np * 4, dd, c.stream));
    }
  }
  if ((st = alloc_match_buffers(c, true))) return st;
  // ---- local fused pass (K9 + cross-stage reduce + deferred stage 2), job-wide ids / windows
  if ((st = alloc_detect(c)) || (st = alloc_localize(c))) return st;
  CK(c.dlate.ensure((uint64_t)c.n_ftiles * ((c.FR + 31) / 32) * 4 + 4));
  queue_fill(c, c.dlate.p, (uint64_t)c.n_ftiles * ((c.FR + 31) / 32) * 4 + 4, 0);
  CK(c.dinfo.ensure((uint64_t)c.n_ftiles * 16 + 16));
  const uint64_t items = (uint64_t)c.NW * W, nlk = (uint64_t)c.NW * np, ncl = (uint64_t)c.TP * c.PP;
  queue_fill(c, c.wd_total.p, items * 4, 0);
  queue_fill(c, c.wd_slow.p, items * 4, 0);
  mark("tables");
  c.launches += timed(c, "k_class_counts", [&] { return launch_class_counts(c); });
  c.launches += timed(c, "k_p2p_roles", [&] { return launch_p2p_roles(c); });
  c.launches += timed(c, stage_active(c) ? "k_stage" : "k_fused", [&] { return launch_fused(c); });
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
    flush_fills(c);
    if (!smap.empty()) {
      k_link_pack<<<(unsigned)smap.size(), 256, 0, c.stream>>>(c.lk_sendmap.as<LinkMap>(), c.inst_rec.as<uint4>(),
                                                              c.slots.as<uint4>(), c.p2p_inst0, c.p2p_slot0,
                                                              c.x_send.as<uint32_t>());
      c.launches += 1;
    }
    int xr = 0;
    timed(c, "x3_alltoall", [&] {
      xch_group_start(c);
      for (uint32_t d = 0; d < G; ++d) {
        if (d == g) continue;
        if (scount[d]) xch_send(c, c.x_send.as<uint32_t>() + soff[d] * LREC, scount[d] * LREC, (int)d);
        if (rcount[d]) xch_recv(c, c.x_recv.as<uint32_t>() + roff[d] * LREC, rcount[d] * LREC, (int)d);
      }
      xr = xch_group_end(c);
      return 0;
    });
    if (xr) { c.err = std::string("exchange all-to-all: ") + xch_error(xr); return SCAN_E_NCCL; }
    if (!rmap.empty()) {
      k_link_unpack<<<(unsigned)rmap.size(), 256, 0, c.stream>>>(c.lk_recvmap.as<LinkMap>(), c.x_recv.as<uint32_t>(),
                                                                c.inst_rec.as<uint4>(), c.slots.as<uint4>(),
                                                                c.lk_key.as<unsigned long long>(), c.p2p_inst0, c.p2p_slot0);
      c.launches += 1;
    }
  }
  mark("x3enq");
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
    // ---- X4: one grouped all-reduce (sum) of every partial result
    const uint64_t nnz_tot = c.nnz_c + W * PCAP;
    int xr = 0;
    timed(c, "x4_allreduce", [&] {
      xch_group_start(c);
      auto ar = [&](DevBuf& b, uint64_t n, int t) { if (n) xch_allreduce(c, b.p, n, t); };
      ar(c.wd_total, items, XU32); ar(c.wd_slow, items, XU32);
      ar(c.wl_joined, items, XU32); ar(c.wl_late, items, XU32);
      ar(c.lk_n, nlk, XU32); ar(c.lk_medp, nlk, XU32); ar(c.lk_medt, nlk, XU32);
      ar(c.lk_used, nlk, XU8); ar(c.lk_elig, nlk, XU8); ar(c.lk_bw, nlk, XF64);
      ar(c.cl_J, ncl, XU32); ar(c.cl_max, ncl, XU32);
      ar(c.ewc, (uint64_t)c.NW * nnz_tot, XU64); ar(c.rk_sum, 3 * W, XU64);
      ar(c.headtail, (uint64_t)G * W + 16, XU64);
      xr = xch_group_end(c);
      return 0;
    });
    if (xr) { c.err = std::string("exchange all-reduce: ") + xch_error(xr); return SCAN_E_NCCL; }
    mark("x4enq");
  }
  // ---- replicated tail on identical job-wide inputs, enqueued behind X4 without a host round trip:
  // the X4 status words go to pinned memory and are checked after the final read-back
  if (!c.h_e) CK(cudaMallocHost(&c.h_e, 16 * sizeof(unsigned long long)));
  CK(cudaMemcpyAsync(c.h_e, ht + (uint64_t)G * W, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c.stream));
  {
    Counters z = c.hc;
    z.n_compared = z.n_slow = z.n_candidates = z.n_class_mismatch = 0;
    z.n_link_slow = z.n_roots = z.n_victims = z.n_unattributed = 0;
    for (auto& v : z.v_count) v = 0;
    CK(cudaMemcpyAsync(c.counters.p, &z, sizeof(Counters), cudaMemcpyHostToDevice, c.stream));
    k_x4_apply<<<1, 32, 0, c.stream>>>(ht + (uint64_t)G * W, c.counters.as<Counters>());
    c.launches += 1;
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
  mark("end");
  const unsigned long long* e = static_cast<const unsigned long long*>(c.h_e);
  if (e[0]) { c.err = "sharded analysis needs an SPMD trace on every shard (fused-pass verification failed)"; return SCAN_E_UNSUPPORTED; }
  if (e[1]) { c.err = "a DP class has unequal compute counts inside a shard other than the last"; return SCAN_E_UNSUPPORTED; }
  if (c.hc.overflow & 24u) {
    c.err = "capacity exceeded: more than 16384 samples on a link / links in a direction class";
    return SCAN_E_UNSUPPORTED;
  }
  c.matched = c.detected = c.localized = true;
  c.fused_used = true;
  c.xwait_pending = true;
  return SCAN_OK;
}

int launch_shard_head(Ctx& c, unsigned long long* out) {
  k_shard_head<<<(unsigned)((c.W + 7) / 8), 256, 0, c.stream>>>(
      c.W, c.rank_off.as<uint64_t>(), c.d_kind, c.r_comm_off.as<uint64_t>(), c.r_bits_off.as<uint64_t>(),
      c.r_ncomp.as<uint32_t>(), c.bits.as<uint32_t>(), c.inst_c.as<uint32_t>(), c.inst_rec.as<uint4>(),
      c.lcfg.stage2_classes, (unsigned long long)c.lcfg.late_margin_ns, c.dcfg.window_iters, c.it_off, out);
  return 1;
}

int launch_shard_fixup(Ctx& c, int G, const unsigned long long* ht) {
  k_shard_fixup<<<(unsigned)((c.W + 255) / 256), 256, 0, c.stream>>>(c.W, G, ht, c.wl_joined.as<uint32_t>(), c.wl_late.as<uint32_t>());
  return 1;
}

void shard_release(Ctx& c) {
  if (c.nccl) ncclCommDestroy((ncclComm_t)c.nccl);
  c.nccl = nullptr;
  if (c.h_pin) cudaFreeHost(c.h_pin);
  c.h_pin = nullptr; c.h_pin_cap = 0;
  if (c.h_e) cudaFreeHost(c.h_e);
  c.h_e = nullptr;
  if (c.ev_x1) { cudaEventDestroy(c.ev_x1); cudaEventDestroy(c.ev_x2); }
  c.ev_x1 = c.ev_x2 = nullptr;
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
