// oracle.cpp — plain, slow, single-threaded CPU reference of MegaScan's analysis pass.
//
// *** TEST INFRASTRUCTURE. *** Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library. The product path
// (paper_2507_19845_b200/) never calls it and shares no code, header or table with it.
//
// It follows PAPER.md §3.2 step by step, with the readings listed in
// DESIGN.md §"Readings" (= SURVEY.md §8(c) table, items 1-20), written in the
// order of SURVEY.md §8(c) "Procedure" O1..O11. Containers are std::map / std::vector,
// medians are full std::sort, every decision is integer or exact-rational arithmetic.
//
// Pins (tests/test_oracle_*.py, -m "not gpu"): SPEC.md examples (S:L202-213,
// S:L336-365), brute-force enumeration of match sets on tiny traces, DES ground
// truth (instance partition, closed-form waits, injected faults), clock-skew
// invariance, stage-1 monotonicity.  The A7-A8 walk has no paper pin: its
// definition is ours (reading R17) and is pinned by hand-built chains.

#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <vector>
#include <string>
#include <algorithm>
#include <tuple>

namespace {

enum { KIND_COMPUTE = 0, KIND_ALLREDUCE = 1, KIND_ALLGATHER = 2, KIND_REDUCESCATTER = 3,
       KIND_BROADCAST = 4, KIND_SEND = 5, KIND_RECV = 6 };
const uint32_t NONE32 = 0xFFFFFFFFu;

// verdicts, labels
enum { V_NONE = 0, V_COMPUTE_SLOW = 1, V_LINK_SLOW = 2, V_BOTH = 3, V_EXONERATED = 4, V_INSUFFICIENT = 5 };
enum { L_CLEAN = 0, L_SOURCE_RANK = 1, L_SOURCE_LINK = 2, L_VICTIM = 3, L_UNATTRIBUTED = 4 };
enum { F_COMPLETE = 1, F_KIND_OK = 2, F_PAYLOAD_OK = 4, F_VALID = 8, F_UNIQUE_LAST = 16, F_WARMUP = 32 };

struct Result {
  int32_t status = 0;
  uint64_t bad_event = ~0ull;
  uint64_t n_instances = 0, n_incomplete = 0, n_kind_mismatch = 0, n_payload_mismatch = 0;
  uint64_t n_windows = 1, n_iters = 0, n_channels = 0, n_links = 0, n_edges = 0;
  std::vector<uint32_t> ev_inst, ev_wait, ev_ref;
  std::vector<uint8_t> ev_slow;
  std::vector<uint8_t> ch_kind; std::vector<uint32_t> ch_a, ch_b, ch_nmem, ch_nmax, ch_nmin; std::vector<uint64_t> ch_base;
  std::vector<uint32_t> in_channel, in_k, in_dmin, in_dmax, in_last, in_npresent, in_payload; std::vector<uint8_t> in_flags;
  std::vector<uint64_t> rk_sum_compute, rk_sum_wait, rk_sum_transfer;
  std::vector<uint32_t> cl_J; std::vector<uint8_t> cl_mismatch;
  std::vector<uint32_t> wd_total, wd_slow; std::vector<uint8_t> wd_cand; std::vector<double> wd_frac;
  std::vector<uint32_t> wl_joined, wl_late; std::vector<double> wl_late_frac; std::vector<uint8_t> wl_verdict, wl_link_slow;
  std::vector<uint32_t> lk_window, lk_src, lk_dst, lk_n, lk_med_payload, lk_med_transfer;
  std::vector<uint8_t> lk_used_warm, lk_slow, lk_dir, lk_eligible; std::vector<double> lk_med_bw;
  std::vector<uint8_t> lb_label, lb_root_kind; std::vector<uint32_t> lb_root_rank, lb_root_src, lb_depth; std::vector<uint64_t> lb_total_wait;
  std::vector<uint32_t> eg_window, eg_src, eg_dst; std::vector<uint64_t> eg_weight;
  std::vector<uint64_t> scalars;
  // NEXT-1 timeline alignment (orc_run_align)
  std::vector<int64_t> al_start; std::vector<int32_t> al_level; std::vector<uint32_t> al_nanchor;
  std::vector<uint64_t> al_residual;
  std::vector<uint64_t> bl_root, bl_inflicted, bl_self, bl_unattributed, bl_suffered;
  uint64_t bl_n_waiting = 0, bl_n_cyclic = 0;
  int32_t al_status = 0;
};

}  // namespace

extern "C" {

typedef struct {
  int32_t tp, pp, dp, pad;
  uint64_t n_events;
  const uint64_t* rank_offsets;  // [W+1]
  const uint32_t* dur;
  const uint16_t* kind_op;
  const uint16_t* meta;
  const uint32_t* comm;
  const uint32_t* payload;
  uint32_t n_comms, pad2;
  const uint64_t* comm_offsets;  // [n_comms+1]
  const uint32_t* comm_members;  // ascending per comm
} orc_input;

typedef struct {
  uint32_t slow_num, slow_den;   // slow iff slow_den*dur > slow_num*ref   (default 3/2)
  uint64_t slow_margin_ns;       // ... and dur - ref > margin             (default 50 us)
  uint32_t cand_num, cand_den;   // candidate iff cand_den*slow > cand_num*total (3/10)
  uint32_t min_samples;          // 10
  uint32_t late_num, late_den;   // ComputeSlow iff late_den*late >= late_num*joined (7/10)
  uint64_t late_margin_ns;       // 100 us
  uint32_t bw_num, bw_den;       // LinkSlow iff bw_den*p_l*t_g < bw_num*p_g*t_l (7/10)
  uint64_t wait_margin_ns;       // 100 us
  uint32_t window_iters;         // 0 = whole trace
  uint32_t stage2_classes;       // bit0 TP, bit1 DP
  uint32_t stage2_mode;          // 0 CONDITIONAL, 1 UNCONDITIONAL
  uint32_t pad;
} orc_config;

}  // extern "C"

namespace {

struct Event { int rank; uint64_t idx; };

// O1 channel key: (0, comm, 0) for collectives, (1, src, dst) for P2P.
typedef std::tuple<int, uint32_t, uint32_t> ChanKey;

struct Oracle {
  const orc_input& in;
  const orc_config& cfg;
  Result& R;
  int W, TP, PP, DP;

  Oracle(const orc_input& i, const orc_config& c, Result& r) : in(i), cfg(c), R(r) {
    TP = in.tp; PP = in.pp; DP = in.dp; W = TP * PP * DP;
  }

  int kind(uint64_t e) const { return in.kind_op[e] & 7; }
  bool iter_end(uint64_t e) const { return (in.kind_op[e] >> 3) & 1; }
  uint32_t op_id(uint64_t e) const { return in.kind_op[e] >> 4; }
  bool warm(uint64_t e) const { return (in.meta[e] >> 14) & 1; }
  int tp_of(int r) const { return r % TP; }
  int dp_of(int r) const { return (r / TP) % DP; }
  int pp_of(int r) const { return r / (TP * DP); }
  int rank_of(int t, int d, int s) const { return t + TP * (d + DP * s); }

  std::vector<uint32_t> members(uint32_t c) const {
    return std::vector<uint32_t>(in.comm_members + in.comm_offsets[c], in.comm_members + in.comm_offsets[c + 1]);
  }

  int run() {
    const uint64_t N = in.n_events;
    // ---- schema validation (SPEC S:L136 parse/schema errors; S:L34, S:L53 invariants) ----
    for (uint32_t c = 0; c < in.n_comms; ++c)
      if (in.comm_offsets[c + 1] < in.comm_offsets[c]) return -1;
    for (int r = 0; r < W; ++r) {
      if (in.rank_offsets[r + 1] < in.rank_offsets[r]) return -1;
      for (uint64_t e = in.rank_offsets[r]; e < in.rank_offsets[r + 1]; ++e) {
        int k = kind(e);
        bool bad = false;
        if (k > KIND_RECV) bad = true;
        else if (k >= KIND_ALLREDUCE && k <= KIND_BROADCAST) {
          if (in.comm[e] >= in.n_comms) bad = true;
          else { auto m = members(in.comm[e]); if (!std::binary_search(m.begin(), m.end(), (uint32_t)r)) bad = true; }
        } else if (k == KIND_SEND || k == KIND_RECV) {
          if (in.comm[e] >= (uint32_t)W || in.comm[e] == (uint32_t)r) bad = true;
        }
        if (bad) { R.bad_event = e; return -2; }
      }
    }

    // ---- iteration index per event (DESIGN reading R18): #iter_end marks before e on its rank ----
    std::vector<uint32_t> iter(N, 0);
    uint64_t n_iters = 0;
    for (int r = 0; r < W; ++r) {
      uint32_t it = 0;
      for (uint64_t e = in.rank_offsets[r]; e < in.rank_offsets[r + 1]; ++e) {
        iter[e] = it;
        if (iter_end(e)) ++it;
        n_iters = std::max<uint64_t>(n_iters, (uint64_t)iter[e] + 1);
      }
    }
    R.n_iters = n_iters;
    uint64_t NW = cfg.window_iters ? std::max<uint64_t>(1, (n_iters + cfg.window_iters - 1) / cfg.window_iters) : 1;
    R.n_windows = NW;
    auto win = [&](uint64_t e) -> uint64_t { return cfg.window_iters ? iter[e] / cfg.window_iters : 0; };

    // ---- O1/O2: channel of every comm event, per-rank occurrence index k ----
    // ("a single pass over the events then matches"; per-communicator
    //  counter = reading R2; FIFO per directed (src,dst) pair = reading R4)
    std::vector<ChanKey> key(N);
    std::vector<uint32_t> kk(N, NONE32);
    std::map<std::pair<int, ChanKey>, uint32_t> cnt;  // (rank, channel) -> count
    std::set<ChanKey> p2p_channels;
    for (int r = 0; r < W; ++r)
      for (uint64_t e = in.rank_offsets[r]; e < in.rank_offsets[r + 1]; ++e) {
        int k = kind(e);
        if (k == KIND_COMPUTE) continue;
        ChanKey ck;
        if (k == KIND_SEND) ck = ChanKey(1, (uint32_t)r, in.comm[e]);
        else if (k == KIND_RECV) ck = ChanKey(1, in.comm[e], (uint32_t)r);
        else ck = ChanKey(0, in.comm[e], 0);
        if (std::get<0>(ck) == 1) p2p_channels.insert(ck);
        key[e] = ck;
        kk[e] = cnt[{r, ck}]++;
      }

    // ---- O3/O4: completeness and instance ids ----
    // channel order: every comm of the table by id, then P2P channels by (src,dst)
    std::vector<ChanKey> chans;
    for (uint32_t c = 0; c < in.n_comms; ++c) chans.push_back(ChanKey(0, c, 0));
    for (auto& ck : p2p_channels) chans.push_back(ck);
    std::map<ChanKey, uint32_t> chan_index;
    for (size_t i = 0; i < chans.size(); ++i) chan_index[chans[i]] = (uint32_t)i;
    std::vector<std::vector<uint32_t>> chan_members(chans.size());
    std::vector<uint32_t> nmax(chans.size()), nmin(chans.size());
    std::vector<uint64_t> base(chans.size());
    uint64_t acc = 0;
    for (size_t i = 0; i < chans.size(); ++i) {
      const ChanKey& ck = chans[i];
      if (std::get<0>(ck) == 0) chan_members[i] = members(std::get<1>(ck));
      else chan_members[i] = {std::get<1>(ck), std::get<2>(ck)};  // slot 0 = src, slot 1 = dst
      uint32_t mx = 0, mn = NONE32;
      for (uint32_t m : chan_members[i]) {
        auto it = cnt.find({(int)m, ck});
        uint32_t c = it == cnt.end() ? 0 : it->second;
        mx = std::max(mx, c); mn = std::min(mn, c);
      }
      if (chan_members[i].empty()) mn = 0;
      nmax[i] = mx; nmin[i] = mn; base[i] = acc; acc += mx;
    }
    if (acc >= NONE32) return -8;  // instance ids must fit u32
    const uint64_t NI = acc;
    R.n_instances = NI; R.n_channels = chans.size();
    R.ch_kind.resize(chans.size()); R.ch_a.resize(chans.size()); R.ch_b.resize(chans.size());
    R.ch_nmem.resize(chans.size()); R.ch_nmax = nmax; R.ch_nmin = nmin; R.ch_base = base;
    for (size_t i = 0; i < chans.size(); ++i) {
      R.ch_kind[i] = (uint8_t)std::get<0>(chans[i]);
      R.ch_a[i] = std::get<1>(chans[i]);
      R.ch_b[i] = std::get<0>(chans[i]) ? std::get<2>(chans[i]) : NONE32;
      R.ch_nmem[i] = (uint32_t)chan_members[i].size();
    }

    // instance -> member events (slot-indexed)
    R.ev_inst.assign(N, NONE32);
    std::map<uint64_t, std::map<uint32_t, uint64_t>> inst_members;  // inst -> slot -> event
    for (int r = 0; r < W; ++r)
      for (uint64_t e = in.rank_offsets[r]; e < in.rank_offsets[r + 1]; ++e) {
        if (kind(e) == KIND_COMPUTE) continue;
        uint32_t ci = chan_index[key[e]];
        uint64_t id = base[ci] + kk[e];
        R.ev_inst[e] = (uint32_t)id;
        const auto& mem = chan_members[ci];
        uint32_t slot;
        if (std::get<0>(key[e]) == 1) slot = (kind(e) == KIND_SEND) ? 0 : 1;
        else slot = (uint32_t)(std::lower_bound(mem.begin(), mem.end(), (uint32_t)r) - mem.begin());
        inst_members[id][slot] = e;
      }

    // ---- O5/O6: integrity and timing decomposition ("logically finish at the same
    // moment" applied per instance = reading R5; wait/transfer = reading R6) ----
    R.in_channel.resize(NI); R.in_k.resize(NI); R.in_dmin.assign(NI, 0); R.in_dmax.assign(NI, 0);
    R.in_last.assign(NI, NONE32); R.in_npresent.assign(NI, 0); R.in_payload.assign(NI, 0); R.in_flags.assign(NI, 0);
    R.ev_wait.assign(N, 0);
    R.rk_sum_compute.assign(W, 0); R.rk_sum_wait.assign(W, 0); R.rk_sum_transfer.assign(W, 0);
    std::vector<uint8_t> inst_cls(NI, 0);  // stage-2 class: 1 TP, 2 DP, 0 other
    for (size_t ci = 0; ci < chans.size(); ++ci) {
      uint8_t cls = 0;
      if (std::get<0>(chans[ci]) == 0) cls = comm_class(chan_members[ci]);
      for (uint32_t k = 0; k < nmax[ci]; ++k) {
        uint64_t id = base[ci] + k;
        R.in_channel[id] = (uint32_t)ci; R.in_k[id] = k; inst_cls[id] = cls;
        auto& sl = inst_members[id];
        R.in_npresent[id] = (uint32_t)sl.size();
        bool is_p2p = std::get<0>(chans[ci]) == 1;
        if (is_p2p) {
          if (sl.count(0)) R.in_payload[id] = in.payload[sl[0]];
          else if (sl.count(1)) R.in_payload[id] = in.payload[sl[1]];
          if (sl.count(0) && warm(sl[0])) R.in_flags[id] |= F_WARMUP;
        }
        bool complete = k < nmin[ci];
        if (!complete) { ++R.n_incomplete; continue; }
        uint8_t f = F_COMPLETE;
        bool kind_ok = true, pay_ok = true;
        int k0 = kind(sl.begin()->second);
        for (auto& p : sl) if (kind(p.second) != k0 && !is_p2p) kind_ok = false;
        if (is_p2p && in.payload[sl[0]] != in.payload[sl[1]]) pay_ok = false;
        if (kind_ok) f |= F_KIND_OK; else ++R.n_kind_mismatch;
        if (pay_ok) f |= F_PAYLOAD_OK; else ++R.n_payload_mismatch;
        if (kind_ok && pay_ok) {
          f |= F_VALID;
          uint32_t dmin = NONE32, dmax = 0;
          for (auto& p : sl) { dmin = std::min(dmin, in.dur[p.second]); dmax = std::max(dmax, in.dur[p.second]); }
          uint32_t last_slot = NONE32, n_at_min = 0;
          for (auto& p : sl) if (in.dur[p.second] == dmin) { if (last_slot == NONE32) last_slot = p.first; ++n_at_min; }
          if (n_at_min == 1) f |= F_UNIQUE_LAST;
          R.in_dmin[id] = dmin; R.in_dmax[id] = dmax;
          R.in_last[id] = chan_members[ci][last_slot];
          for (auto& p : sl) {
            uint64_t e = p.second;
            R.ev_wait[e] = in.dur[e] - dmin;
          }
        }
        R.in_flags[id] |= f;
      }
    }
    for (int r = 0; r < W; ++r)
      for (uint64_t e = in.rank_offsets[r]; e < in.rank_offsets[r + 1]; ++e) {
        if (kind(e) == KIND_COMPUTE) { R.rk_sum_compute[r] += in.dur[e]; continue; }
        uint32_t id = R.ev_inst[e];
        if (R.in_flags[id] & F_VALID) { R.rk_sum_wait[r] += R.ev_wait[e]; R.rk_sum_transfer[r] += R.in_dmin[id]; }
      }

    // ---- O7: stage 1, cross-DP comparison of identical kernels ----
    // peer class (tp,pp); position j among compute ops; leave-one-out lower median of
    // the other DP peers (reading R8); common prefix of equal op ids (reading R9).
    R.ev_slow.assign(N, 0); R.ev_ref.assign(N, NONE32);
    R.wd_total.assign(NW * W, 0); R.wd_slow.assign(NW * W, 0); R.wd_cand.assign(NW * W, 0); R.wd_frac.assign(NW * W, 0.0);
    R.cl_J.assign((size_t)TP * PP, 0); R.cl_mismatch.assign((size_t)TP * PP, 0);
    std::vector<std::vector<uint64_t>> comp(W);  // compute events per rank, program order
    for (int r = 0; r < W; ++r)
      for (uint64_t e = in.rank_offsets[r]; e < in.rank_offsets[r + 1]; ++e)
        if (kind(e) == KIND_COMPUTE) comp[r].push_back(e);
    if (DP >= 2) {
      for (int s = 0; s < PP; ++s)
        for (int t = 0; t < TP; ++t) {
          std::vector<int> peers;
          for (int d = 0; d < DP; ++d) peers.push_back(rank_of(t, d, s));
          size_t mincnt = SIZE_MAX, maxcnt = 0;
          for (int p : peers) { mincnt = std::min(mincnt, comp[p].size()); maxcnt = std::max(maxcnt, comp[p].size()); }
          size_t J = mincnt;
          for (size_t j = 0; j < mincnt && J == mincnt; ++j)
            for (int p : peers) if (op_id(comp[p][j]) != op_id(comp[peers[0]][j])) { J = j; break; }
          R.cl_J[(size_t)s * TP + t] = (uint32_t)J;
          R.cl_mismatch[(size_t)s * TP + t] = (J != maxcnt) ? 1 : 0;
          for (size_t j = 0; j < J; ++j)
            for (size_t i = 0; i < peers.size(); ++i) {
              std::vector<uint32_t> others;
              for (size_t q = 0; q < peers.size(); ++q) if (q != i) others.push_back(in.dur[comp[peers[q]][j]]);
              std::sort(others.begin(), others.end());
              uint32_t ref = others[(others.size() - 1) / 2];   // lower median (reading R15)
              uint64_t e = comp[peers[i]][j];
              uint64_t dur = in.dur[e];
              bool slow = (uint64_t)cfg.slow_den * dur > (uint64_t)cfg.slow_num * ref && dur > (uint64_t)ref + cfg.slow_margin_ns;
              R.ev_ref[e] = ref;
              R.ev_slow[e] = slow ? 1 : 0;
              uint64_t w = win(e) * W + peers[i];
              R.wd_total[w] += 1;
              R.wd_slow[w] += slow ? 1 : 0;
            }
        }
    }
    for (uint64_t w = 0; w < NW * W; ++w) {
      R.wd_cand[w] = (R.wd_total[w] >= cfg.min_samples &&
                      (uint64_t)cfg.cand_den * R.wd_slow[w] > (uint64_t)cfg.cand_num * R.wd_total[w]) ? 1 : 0;
      R.wd_frac[w] = R.wd_total[w] ? (double)R.wd_slow[w] / (double)R.wd_total[w] : 0.0;
    }

    // ---- O8: stage 2, start lag within TP and DP collectives ----
    // late iff r is the unique last arriver and dmax - dmin > margin (readings R11, R20);
    // counted over instances whose preceding compute segment has a slow op (CONDITIONAL).
    R.wl_joined.assign(NW * W, 0); R.wl_late.assign(NW * W, 0); R.wl_late_frac.assign(NW * W, 0.0);
    R.wl_verdict.assign(NW * W, V_NONE); R.wl_link_slow.assign(NW * W, 0);
    for (int r = 0; r < W; ++r) {
      bool seg_slow = false;  // OR of slow bits since the previous comm event
      for (uint64_t e = in.rank_offsets[r]; e < in.rank_offsets[r + 1]; ++e) {
        if (kind(e) == KIND_COMPUTE) { if (R.ev_slow[e]) seg_slow = true; continue; }
        bool pslow = seg_slow;
        seg_slow = false;
        uint32_t id = R.ev_inst[e];
        if (!(R.in_flags[id] & F_VALID)) continue;
        uint8_t cls = inst_cls[id];
        if (cls == 0 || !((cfg.stage2_classes >> (cls - 1)) & 1)) continue;
        if (cfg.stage2_mode == 0 && !pslow) continue;
        uint64_t w = win(e) * W + r;
        R.wl_joined[w] += 1;
        if ((R.in_flags[id] & F_UNIQUE_LAST) && R.in_last[id] == (uint32_t)r &&
            (uint64_t)(R.in_dmax[id] - R.in_dmin[id]) > cfg.late_margin_ns)
          R.wl_late[w] += 1;
      }
    }

    // ---- O9: stage 3, P2P effective bandwidth ----
    // bw = payload / transfer, transfer = dmin (reading R7); warm-up samples if >= min_samples
    // (reading R13); lower median under exact ratio order; LinkSlow vs the lower median of
    // same-direction link medians (reading R14).
    std::vector<uint32_t> p2p_ci;
    for (size_t ci = 0; ci < chans.size(); ++ci) if (std::get<0>(chans[ci]) == 1) p2p_ci.push_back((uint32_t)ci);
    const size_t NL = p2p_ci.size();
    R.n_links = NW * NL;
    R.lk_window.resize(NW * NL); R.lk_src.resize(NW * NL); R.lk_dst.resize(NW * NL);
    R.lk_n.assign(NW * NL, 0); R.lk_med_payload.assign(NW * NL, 0); R.lk_med_transfer.assign(NW * NL, 0);
    R.lk_used_warm.assign(NW * NL, 0); R.lk_slow.assign(NW * NL, 0); R.lk_dir.assign(NW * NL, 0);
    R.lk_eligible.assign(NW * NL, 0); R.lk_med_bw.assign(NW * NL, 0.0);
    // ratio order: a < b  <=>  p_a * t_b < p_b * t_a
    auto ratio_less = [](uint32_t pa, uint32_t ta, uint32_t pb, uint32_t tb) {
      return (unsigned __int128)pa * tb < (unsigned __int128)pb * ta;
    };
    for (uint64_t w = 0; w < NW; ++w)
      for (size_t l = 0; l < NL; ++l) {
        uint32_t ci = p2p_ci[l];
        size_t o = w * NL + l;
        uint32_t src = std::get<1>(chans[ci]), dst = std::get<2>(chans[ci]);
        R.lk_window[o] = (uint32_t)w; R.lk_src[o] = src; R.lk_dst[o] = dst;
        int dpp = pp_of((int)dst) - pp_of((int)src);
        R.lk_dir[o] = dpp == 1 ? 0 : (dpp == -1 ? 1 : 2);
        struct S { uint32_t p, t, id; bool warm; };
        std::vector<S> all, warmv;
        for (uint32_t k = 0; k < nmax[ci]; ++k) {
          uint64_t id = base[ci] + k;
          if (!(R.in_flags[id] & F_VALID)) continue;
          uint64_t se = inst_members[id][0];  // SEND event decides the window and the warm-up flag
          if (win(se) != w) continue;
          if (R.in_dmin[id] == 0) continue;  // non-positive latency: discarded
          S smp{R.in_payload[id], R.in_dmin[id], (uint32_t)id, (R.in_flags[id] & F_WARMUP) != 0};
          all.push_back(smp);
          if (smp.warm) warmv.push_back(smp);
        }
        std::vector<S>& use = warmv.size() >= cfg.min_samples ? warmv : all;
        R.lk_used_warm[o] = warmv.size() >= cfg.min_samples ? 1 : 0;
        R.lk_n[o] = (uint32_t)use.size();
        if (use.empty()) continue;
        std::sort(use.begin(), use.end(), [&](const S& a, const S& b) {
          if (ratio_less(a.p, a.t, b.p, b.t)) return true;
          if (ratio_less(b.p, b.t, a.p, a.t)) return false;
          return a.id < b.id;
        });
        const S& m = use[(use.size() - 1) / 2];
        R.lk_med_payload[o] = m.p; R.lk_med_transfer[o] = m.t;
        R.lk_med_bw[o] = (double)m.p / (double)m.t;
        R.lk_eligible[o] = use.size() >= cfg.min_samples ? 1 : 0;
      }
    for (uint64_t w = 0; w < NW; ++w)
      for (int dir = 0; dir < 3; ++dir) {
        std::vector<size_t> links;
        for (size_t l = 0; l < NL; ++l) { size_t o = w * NL + l; if (R.lk_eligible[o] && R.lk_dir[o] == dir) links.push_back(o); }
        if (links.empty()) continue;
        std::sort(links.begin(), links.end(), [&](size_t a, size_t b) {
          if (ratio_less(R.lk_med_payload[a], R.lk_med_transfer[a], R.lk_med_payload[b], R.lk_med_transfer[b])) return true;
          if (ratio_less(R.lk_med_payload[b], R.lk_med_transfer[b], R.lk_med_payload[a], R.lk_med_transfer[a])) return false;
          return a < b;  // (src,dst) order within a window
        });
        size_t g = links[(links.size() - 1) / 2];
        unsigned __int128 pg = R.lk_med_payload[g], tg = R.lk_med_transfer[g];
        for (size_t o : links) {
          unsigned __int128 pl = R.lk_med_payload[o], tl = R.lk_med_transfer[o];
          if ((unsigned __int128)cfg.bw_den * pl * tg < (unsigned __int128)cfg.bw_num * pg * tl) {
            R.lk_slow[o] = 1;
            R.wl_link_slow[w * W + R.lk_src[o]] = 1;  // attributed to the egress rank (reading R14)
          }
        }
      }

    // ---- verdicts (ComputeSlow / LinkSlow / Both; candidates failing stage 2 exonerated) ----
    for (uint64_t w = 0; w < NW * W; ++w) {
      R.wl_late_frac[w] = R.wl_joined[w] ? (double)R.wl_late[w] / (double)R.wl_joined[w] : 0.0;
      int v = V_NONE;
      if (R.wd_cand[w]) {
        if (R.wl_joined[w] < cfg.min_samples) v = V_INSUFFICIENT;
        else if ((uint64_t)cfg.late_den * R.wl_late[w] >= (uint64_t)cfg.late_num * R.wl_joined[w]) v = V_COMPUTE_SLOW;
        else v = V_EXONERATED;
      }
      if (R.wl_link_slow[w]) v = (v == V_COMPUTE_SLOW) ? V_BOTH : V_LINK_SLOW;
      R.wl_verdict[w] = (uint8_t)v;
    }

    // ---- O10: wait-for edges and the source/victim walk (reading R17) ----
    std::map<std::tuple<uint64_t, uint32_t, uint32_t>, uint64_t> edges;  // (window, waiter, waited-on)
    for (uint64_t id = 0; id < NI; ++id) {
      if (!(R.in_flags[id] & F_VALID)) continue;
      for (auto& p : inst_members[id]) {
        uint64_t e = p.second;
        uint32_t rm = chan_members[R.in_channel[id]][p.first];
        if (rm == R.in_last[id]) continue;
        if ((uint64_t)R.ev_wait[e] > cfg.wait_margin_ns) edges[std::make_tuple(win(e), rm, R.in_last[id])] += R.ev_wait[e];
      }
    }
    R.n_edges = edges.size();
    for (auto& x : edges) {
      R.eg_window.push_back((uint32_t)std::get<0>(x.first)); R.eg_src.push_back(std::get<1>(x.first));
      R.eg_dst.push_back(std::get<2>(x.first)); R.eg_weight.push_back(x.second);
    }
    R.lb_label.assign(NW * W, L_CLEAN); R.lb_root_kind.assign(NW * W, 0); R.lb_root_rank.assign(NW * W, NONE32);
    R.lb_root_src.assign(NW * W, NONE32); R.lb_depth.assign(NW * W, 0); R.lb_total_wait.assign(NW * W, 0);
    for (auto& x : edges) R.lb_total_wait[std::get<0>(x.first) * W + std::get<1>(x.first)] += x.second;
    for (uint64_t w = 0; w < NW; ++w) {
      std::vector<int> level(W, -1);
      int n_roots = 0;
      for (int r = 0; r < W; ++r) {
        int v = R.wl_verdict[w * W + r];
        if (v == V_COMPUTE_SLOW || v == V_BOTH) {
          level[r] = 0; ++n_roots;
          R.lb_label[w * W + r] = L_SOURCE_RANK; R.lb_root_kind[w * W + r] = 1;
          R.lb_root_rank[w * W + r] = (uint32_t)r; R.lb_root_src[w * W + r] = (uint32_t)r;
        }
      }
      for (size_t l = 0; l < NL; ++l) {  // ascending (src,dst): the lowest LinkSlow in-link wins
        size_t o = w * NL + l;
        if (!R.lk_slow[o]) continue;
        uint32_t d = R.lk_dst[o];
        if (level[d] >= 0) continue;
        level[d] = 0; ++n_roots;
        R.lb_label[w * W + d] = L_SOURCE_LINK; R.lb_root_kind[w * W + d] = 2;
        R.lb_root_rank[w * W + d] = d; R.lb_root_src[w * W + d] = R.lk_src[o];
      }
      // out-edges of each rank in this window
      std::vector<std::vector<std::pair<uint32_t, uint64_t>>> out(W);
      for (auto& x : edges) if (std::get<0>(x.first) == w) out[std::get<1>(x.first)].push_back({std::get<2>(x.first), x.second});
      for (int d = 0;; ++d) {
        std::vector<std::pair<int, int>> newly;  // (rank, chosen neighbour)
        for (int u = 0; u < W; ++u) {
          if (level[u] >= 0) continue;
          int best = -1; uint64_t bw = 0;
          for (auto& nb : out[u]) {
            if (level[nb.first] != d) continue;
            if (best < 0 || nb.second > bw || (nb.second == bw && (int)nb.first < best)) { best = (int)nb.first; bw = nb.second; }
          }
          if (best >= 0) newly.push_back({u, best});
        }
        if (newly.empty()) break;
        for (auto& p : newly) {
          int u = p.first, v = p.second;
          level[u] = d + 1;
          R.lb_label[w * W + u] = L_VICTIM;
          R.lb_root_kind[w * W + u] = R.lb_root_kind[w * W + v];
          R.lb_root_rank[w * W + u] = R.lb_root_rank[w * W + v];
          R.lb_root_src[w * W + u] = R.lb_root_src[w * W + v];
          R.lb_depth[w * W + u] = (uint32_t)(d + 1);
        }
      }
      for (int u = 0; u < W; ++u)
        if (level[u] < 0 && R.lb_total_wait[w * W + u] > 0 && n_roots > 0) R.lb_label[w * W + u] = L_UNATTRIBUTED;
    }
    return (R.n_incomplete || R.n_kind_mismatch || R.n_payload_mismatch) ? 1 : 0;
  }

  // ---- NEXT-1 timeline alignment (members of a synchronous call "logically finish at the
  // same moment"; a reference rank; the others aligned to it "iteratively", anchors at the identified
  // instances; SPEC S:L243-300 ClockMap). Readings (AL1-AL6):
  //   AL1 anchors = ends (start + dur) of a rank's collective events (kinds 1-4) whose instance is
  //       VALID; P2P excluded
  //   AL2 "iteratively" = BFS levels from the reference over "shares a valid collective instance";
  //       level-k ranks use members of levels < k only (one level at a time)
  //   AL3 target of an instance = the maximum aligned end over those members; anchor =
  //       (local end, target - local end), in program order; an end equal to the previous
  //       anchor's is skipped; decreasing candidate ends on a rank -> status -9 (unsupported)
  //   AL4 offset(t): none -> 0; before the first / after the last anchor -> that anchor's offset;
  //       between anchors i, i+1: o_i + floor((o_i+1 - o_i) * (t - t_i) / (t_i+1 - t_i)), exact
  //   AL5 aligned start = start + offset(start); ranks not reached keep their local clock (level -1)
  //   AL6 residual of a rank = max over its anchor candidates of (max aligned end over the
  //       instance's aligned members - its own aligned end)
  static int64_t floor_div(__int128 n, __int128 d) {
    __int128 q = n / d;
    if ((n % d != 0) && ((n < 0) != (d < 0))) q -= 1;
    return (int64_t)q;
  }
  static int64_t offset_at(const std::vector<std::pair<int64_t, int64_t>>& a, int64_t t) {
    if (a.empty()) return 0;
    if (t <= a.front().first) return a.front().second;
    if (t >= a.back().first) return a.back().second;
    size_t i = std::upper_bound(a.begin(), a.end(), std::make_pair(t, INT64_MAX)) - a.begin() - 1;  // t_i <= t < t_i+1
    const __int128 o0 = a[i].second, o1 = a[i + 1].second, t0 = a[i].first, t1 = a[i + 1].first;
    return (int64_t)(o0 + floor_div((o1 - o0) * ((__int128)t - t0), t1 - t0));
  }
  int align(const int64_t* start, int ref, std::vector<int64_t>& al_start, std::vector<int32_t>& level,
            std::vector<uint32_t>& nanchor, std::vector<uint64_t>& residual) {
    const uint64_t N = in.n_events;
    al_start.assign(start, start + N);
    level.assign(W, -1); nanchor.assign(W, 0); residual.assign(W, 0);
    if (ref < 0 || ref >= W) return -1;
    std::vector<std::vector<uint64_t>> cand(W);
    std::map<uint32_t, std::vector<std::pair<int, uint64_t>>> inst_ev;  // instance -> (rank, event)
    for (int r = 0; r < W; ++r)
      for (uint64_t e = in.rank_offsets[r]; e < in.rank_offsets[r + 1]; ++e) {
        const int k = kind(e);
        if (k < KIND_ALLREDUCE || k > KIND_BROADCAST) continue;
        const uint32_t id = R.ev_inst[e];
        if (!(R.in_flags[id] & F_VALID)) continue;
        if (!cand[r].empty()) {
          const uint64_t p = cand[r].back();
          if (start[e] + (int64_t)in.dur[e] < start[p] + (int64_t)in.dur[p]) return -9;
        }
        cand[r].push_back(e);
        inst_ev[id].push_back({r, e});
      }
    // BFS levels (AL2)
    std::vector<std::set<int>> adj(W);
    for (auto& kv : inst_ev)
      for (auto& a : kv.second)
        for (auto& b : kv.second)
          if (a.first != b.first) adj[a.first].insert(b.first);
    std::vector<int> order{ref};
    level[ref] = 0;
    for (size_t q = 0; q < order.size(); ++q)
      for (int m : adj[order[q]])
        if (level[m] < 0) { level[m] = level[order[q]] + 1; order.push_back(m); }
    int maxlev = 0;
    for (int r = 0; r < W; ++r) maxlev = std::max(maxlev, level[r]);
    std::vector<int64_t> aend(N, 0);  // event -> aligned end (collective candidates of aligned ranks)
    std::vector<std::vector<std::pair<int64_t, int64_t>>> anc(W);
    for (uint64_t e : cand[ref]) aend[e] = start[e] + (int64_t)in.dur[e];
    for (int k = 1; k <= maxlev; ++k) {
      for (int r = 0; r < W; ++r) {  // AL3: anchors from members of earlier levels
        if (level[r] != k) continue;
        for (uint64_t e : cand[r]) {
          const int64_t t = start[e] + (int64_t)in.dur[e];
          bool have = false;
          int64_t tgt = 0;
          for (auto& m : inst_ev[R.ev_inst[e]])
            if (m.first != r && level[m.first] >= 0 && level[m.first] < k) {
              const int64_t v = aend[m.second];
              if (!have || v > tgt) tgt = v;
              have = true;
            }
          if (have && (anc[r].empty() || t > anc[r].back().first)) anc[r].push_back({t, tgt - t});
        }
      }
      for (int r = 0; r < W; ++r) {
        if (level[r] != k) continue;
        for (uint64_t e : cand[r]) {
          const int64_t t = start[e] + (int64_t)in.dur[e];
          aend[e] = t + offset_at(anc[r], t);
        }
      }
    }
    for (int r = 0; r < W; ++r) {  // AL5, AL6
      nanchor[r] = (uint32_t)anc[r].size();
      if (level[r] < 0) continue;
      for (uint64_t e = in.rank_offsets[r]; e < in.rank_offsets[r + 1]; ++e) al_start[e] = start[e] + offset_at(anc[r], start[e]);
      uint64_t res = 0;
      for (uint64_t e : cand[r]) {
        int64_t fin = INT64_MIN;
        for (auto& m : inst_ev[R.ev_inst[e]]) if (level[m.first] >= 0) fin = std::max(fin, aend[m.second]);
        res = std::max<uint64_t>(res, (uint64_t)(fin - aend[e]));
      }
      residual[r] = res;
    }
    return 0;
  }

  // NEXT-4 event-level blame (readings EB1-EB6; "ranks that merely
  // suffer collateral slowdown will only lag because they are waiting for the faulty peer"):
  // every waiting communication event is traced back through the happens-before structure to the
  // event where its delay began.
  void blame() {
    const uint64_t N = in.n_events;
    const uint64_t NONE = ~0ull, CYCLE = ~0ull - 1;
    std::vector<int> rank(N);
    for (int r = 0; r < W; ++r)
      for (uint64_t e = in.rank_offsets[r]; e < in.rank_offsets[r + 1]; ++e) rank[e] = r;
    // member event of every (instance, rank)
    std::map<std::pair<uint32_t, int>, uint64_t> mev;
    for (uint64_t e = 0; e < N; ++e)
      if (kind(e) != KIND_COMPUTE) mev[{R.ev_inst[e], rank[e]}] = e;
    // EB1: a waiting event is a communication event of a VALID instance with wait > 0
    auto waiting = [&](uint64_t e) {
      return kind(e) != KIND_COMPUTE && (R.in_flags[R.ev_inst[e]] & F_VALID) && R.ev_wait[e] > 0;
    };
    // EB2 / EB3: the pointer of every event
    std::vector<uint64_t> ptr(N);
    for (uint64_t e = 0; e < N; ++e) {
      const bool first = e == in.rank_offsets[rank[e]];
      if (kind(e) == KIND_COMPUTE) ptr[e] = e;                       // a compute event is a root
      else if (waiting(e)) {                                         // delayed by the last arriver's
        const uint32_t id = R.ev_inst[e];                            // previous event
        const uint64_t le = mev.at({id, (int)R.in_last[id]});
        ptr[e] = le == in.rank_offsets[rank[le]] ? le : le - 1;
      } else ptr[e] = first ? e : e - 1;                             // its own rank's previous event
    }
    // EB4: follow the pointers to a fixed point; revisiting an event is a cycle
    R.bl_root.assign(N, NONE);
    R.bl_inflicted.assign(W, 0); R.bl_self.assign(W, 0); R.bl_unattributed.assign(W, 0); R.bl_suffered.assign(W, 0);
    for (uint64_t e = 0; e < N; ++e) {
      if (!waiting(e)) continue;
      ++R.bl_n_waiting;
      std::set<uint64_t> seen;
      uint64_t x = e;
      while (ptr[x] != x) {
        if (!seen.insert(x).second) { x = CYCLE; break; }
        x = ptr[x];
      }
      R.bl_root[e] = x;
      // EB5: the wait is blamed on the root's rank
      const int r = rank[e];
      const uint64_t w = R.ev_wait[e];
      R.bl_suffered[r] += w;
      if (x == CYCLE) { R.bl_unattributed[r] += w; ++R.bl_n_cyclic; }
      else if (rank[x] == r) R.bl_self[r] += w;
      else R.bl_inflicted[rank[x]] += w;
    }
  }

  // stage-2 class of a communicator from the topology (reading R12): 1 = TP group, 2 = DP group
  uint8_t comm_class(const std::vector<uint32_t>& m) const {
    if (TP >= 2 && (int)m.size() == TP) {
      int r0 = (int)m[0];
      if (tp_of(r0) == 0) {
        bool ok = true;
        for (int t = 0; t < TP; ++t) if ((int)m[t] != r0 + t) ok = false;
        if (ok) return 1;
      }
    }
    if (DP >= 2 && (int)m.size() == DP) {
      int r0 = (int)m[0];
      if (dp_of(r0) == 0) {
        bool ok = true;
        for (int d = 0; d < DP; ++d) if ((int)m[d] != rank_of(tp_of(r0), d, pp_of(r0))) ok = false;
        if (ok) return 2;
      }
    }
    return 0;
  }
};

template <class T>
void expose(std::vector<T>& v, void** p, uint64_t* n) { *p = v.data(); *n = v.size() * sizeof(T); }

}  // namespace

extern "C" {

void* orc_run(const orc_input* in, const orc_config* cfg, int32_t* status) {
  Result* R = new Result();
  if (in->tp < 1 || in->pp < 1 || in->dp < 1) { R->status = -1; *status = -1; return R; }
  Oracle o(*in, *cfg, *R);
  R->status = o.run();
  *status = R->status;
  R->scalars = {(uint64_t)(int64_t)R->status, R->bad_event, R->n_instances, R->n_incomplete, R->n_kind_mismatch,
                R->n_payload_mismatch, R->n_windows, R->n_iters, R->n_channels, R->n_links, R->n_edges};
  return R;
}

// run() then the timeline alignment on its instances; *al_status: 0 ok, -1 bad reference,
// -9 decreasing collective end times on a rank
void* orc_run_align(const orc_input* in, const orc_config* cfg, const int64_t* start_ns, int32_t reference,
                    int32_t* status, int32_t* al_status) {
  Result* R = static_cast<Result*>(orc_run(in, cfg, status));
  *al_status = -1;
  if (*status < 0 || !start_ns) return R;
  Oracle o(*in, *cfg, *R);
  R->al_status = o.align(start_ns, reference, R->al_start, R->al_level, R->al_nanchor, R->al_residual);
  *al_status = R->al_status;
  return R;
}

// run() then the event-level blame (NEXT-4) on its instances
void* orc_run_blame(const orc_input* in, const orc_config* cfg, int32_t* status) {
  Result* R = static_cast<Result*>(orc_run(in, cfg, status));
  if (*status < 0) return R;
  Oracle o(*in, *cfg, *R);
  o.blame();
  R->scalars.push_back(R->bl_n_waiting);
  R->scalars.push_back(R->bl_n_cyclic);
  return R;
}

void orc_free(void* h) { delete (Result*)h; }

// Named result arrays; returns 0 if found.
int orc_array(void* h, const char* name, void** ptr, uint64_t* nbytes) {
  Result& R = *(Result*)h;
  std::string n(name);
#define X(field) if (n == #field) { expose(R.field, ptr, nbytes); return 0; }
  X(scalars)
  X(ev_inst) X(ev_wait) X(ev_ref) X(ev_slow)
  X(ch_kind) X(ch_a) X(ch_b) X(ch_nmem) X(ch_nmax) X(ch_nmin) X(ch_base)
  X(in_channel) X(in_k) X(in_dmin) X(in_dmax) X(in_last) X(in_npresent) X(in_payload) X(in_flags)
  X(rk_sum_compute) X(rk_sum_wait) X(rk_sum_transfer)
  X(cl_J) X(cl_mismatch)
  X(wd_total) X(wd_slow) X(wd_cand) X(wd_frac)
  X(wl_joined) X(wl_late) X(wl_late_frac) X(wl_verdict) X(wl_link_slow)
  X(lk_window) X(lk_src) X(lk_dst) X(lk_n) X(lk_med_payload) X(lk_med_transfer) X(lk_used_warm) X(lk_slow)
  X(lk_dir) X(lk_eligible) X(lk_med_bw)
  X(lb_label) X(lb_root_kind) X(lb_root_rank) X(lb_root_src) X(lb_depth) X(lb_total_wait)
  X(eg_window) X(eg_src) X(eg_dst) X(eg_weight)
  X(al_start) X(al_level) X(al_nanchor) X(al_residual)
  X(bl_root) X(bl_inflicted) X(bl_self) X(bl_unattributed) X(bl_suffered)
#undef X
  return -1;
}

}  // extern "C"
