// tracegen — seeded synthetic Megatron-style trace generator (TEST INFRASTRUCTURE).
//
// Shared input source for BOTH the oracle (oracle/) and the CUDA path
// (paper_2507_19845_b200/). It holds none of MegaScan's analysis arithmetic:
// it is a discrete-event simulation (DES) of a TP x PP x DP Megatron job that
// *produces* per-rank CUDA-event traces (§3.2 "Workload tracing",
// P:L105-114) with injectable faults ("GPU down-clocking or link jitter").
//
// Workload model:
//  * rank = tp + TP*(dp + DP*pp)  (TP fastest, then DP, then PP)
//  * non-interleaved 1F1B schedule with Megatron's grouped P2P
//    (send_forward_recv_backward / send_backward_recv_forward).
//  * per layer forward: qkv, attn, proj, TP-AR, fc1, fc2, TP-AR;
//    backward mirrored: fc2_b, fc1_b, TP-AR, proj_b, attn_b, qkv_b, TP-AR.
//  * iteration end: L_s DP grad all-reduces, embedding-group AR (PP>1),
//    model-parallel grad-norm AR, optimizer step (carries the iter_end bit).
//  * collectives: all members wait for the latest arrival, then the
//    collective's own duration; every member's CUDA-event duration
//    is end - own arrival.  P2P pairs are rendezvous: both sides end at
//    max(post) + transfer.  A rank resumes after all ops of its group end.
//  * iterations are separated by a global barrier (the job-level
//    optimizer/timer sync), so iterations simulate independently and in
//    parallel; only start_ns depends on the previous iterations.
//  * jitter: every duration x U[1-j, 1+j], counter-based RNG keyed by
//    (seed, iteration, rank/comm/link, index).
//  * faults: THROTTLE(rank, factor, [it0,it1), prob) scales compute ops;
//    LINK_JITTER(src,dst,[it0,it1)) scales transfer by (1+Exp(1));
//    LINK_DEGRADE(src,dst,factor,[it0,it1)) divides link bandwidth by factor.
//  * clock skew (optional): start_ns = true + offset_r + drift_r * true,
//    offset ~ U[-2ms, 2ms], drift 10 ppm.  Durations are untouched.
//
// Event columns written (SoA, events grouped by rank in program order):
//   start_ns i64, dur_ns u32, kind_op u16 (kind:3 | iter_end:1 | op_id:12),
//   meta u16 (mb:10 | chunk:3 | bwd:1 | warmup:1 | rsv:1),
//   comm u32 (collective: comm id; SEND/RECV: peer rank), payload u32.
// Ground truth (optional): gt_inst u64 per event (DES instance id, UINT64_MAX
// for compute), gt_true_start i64 per event (skew-free start).

#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <thread>
#include <atomic>
#include <algorithm>
#include <cstdio>
#include <string>

extern "C" {

typedef struct gen_fault_c {
  int32_t type, a, b, it0, it1, pad;
  double factor, prob;
} gen_fault_c;

typedef struct gen_config_c {
  int32_t tp, pp, dp, layers_per_stage, microbatches, iterations;
  uint64_t seed;
  int64_t hidden;
  double jitter;
  int32_t clock_skew, n_faults;
  const gen_fault_c* faults;
  int32_t n_threads, it_begin;  // iteration range [it_begin, it_end) to emit; it_end = 0: all iterations
  int32_t it_end, pad;
} gen_config_c;

}

namespace {

enum Kind : uint16_t { K_COMPUTE = 0, K_ALLREDUCE = 1, K_ALLGATHER = 2, K_REDUCESCATTER = 3,
                       K_BROADCAST = 4, K_SEND = 5, K_RECV = 6 };
enum Role : uint8_t { R_TP = 0, R_DP = 1, R_MP = 2, R_EMB = 3 };
enum OpType : uint8_t { OT_COMPUTE = 0, OT_COLL = 1, OT_P2P = 2 };

struct Fault {
  int32_t type;  // 1 throttle, 2 link jitter, 3 link degrade
  int32_t a;     // rank (throttle) or src
  int32_t b;     // dst (link faults)
  int32_t it0, it1;
  double factor;
  double prob;
};

struct P2POp { uint8_t is_send; int8_t dir; uint8_t warmup; uint8_t pad; uint16_t meta; };

struct ProgOp {
  uint8_t type;
  uint8_t role;     // OT_COLL
  uint8_t n_p2p;    // OT_P2P: 1 or 2
  uint8_t pad;
  uint16_t kind_op; // OT_COMPUTE / OT_COLL
  uint16_t meta;
  uint32_t base_dur;
  P2POp p2p[2];
};

inline uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
inline uint64_t rng4(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return splitmix(splitmix(splitmix(splitmix(seed) ^ a) ^ b) ^ c);
}
inline double u01(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

struct Cfg {
  int tp, pp, dp, ls, m, iters;
  uint64_t seed;
  int64_t hidden;
  double jitter;
  int skew;
  std::vector<Fault> faults;
  int threads;
  int it_begin = 0, it_end = 0;  // emitted iteration range (events of iteration it land at it - it_begin)
};

inline uint16_t KO(uint16_t kind, uint16_t op, bool iter_end = false) {
  return (uint16_t)((kind & 7u) | (iter_end ? 8u : 0u) | ((op & 0xFFFu) << 4));
}
inline uint16_t META(int mb, int chunk, int bwd, int warmup) {
  return (uint16_t)((mb & 1023) | ((chunk & 7) << 10) | ((bwd & 1) << 13) | ((warmup & 1) << 14));
}

// compute op codes (op_id = layer*16 + code); codes 0..15
enum { C_QKV = 1, C_ATTN, C_PROJ, C_FC1, C_FC2, C_QKV_B, C_ATTN_B, C_PROJ_B, C_FC1_B, C_FC2_B,
       C_EMB, C_EMB_B, C_LOSS, C_LOSS_B, C_OPT };
// comm op codes (op_id for collectives / p2p), distinct values for readability
enum { O_TP_AR = 1, O_DP_AR = 2, O_MP_AR = 3, O_EMB_AR = 4, O_P2P_ACT = 5, O_P2P_GRAD = 6 };

struct Program {
  std::vector<ProgOp> ops;
  uint32_t n_events = 0;
};

void add_compute(Program& p, int layer, int code, uint32_t dur, int mb, int bwd, bool iter_end = false) {
  ProgOp o{}; o.type = OT_COMPUTE; o.kind_op = KO(K_COMPUTE, (uint16_t)(layer * 16 + code), iter_end);
  o.meta = META(mb, 0, bwd, 0); o.base_dur = dur; p.ops.push_back(o); p.n_events += 1;
}
void add_coll(Program& p, int role, int opcode, uint32_t dur, int mb, int bwd) {
  ProgOp o{}; o.type = OT_COLL; o.role = (uint8_t)role; o.kind_op = KO(K_ALLREDUCE, (uint16_t)opcode);
  o.meta = META(mb, 0, bwd, 0); o.base_dur = dur; p.ops.push_back(o); p.n_events += 1;
}
void add_p2p(Program& p, std::initializer_list<P2POp> ops) {
  ProgOp o{}; o.type = OT_P2P; o.n_p2p = 0;
  for (auto& x : ops) o.p2p[o.n_p2p++] = x;
  p.ops.push_back(o); p.n_events += o.n_p2p;
}

// Base durations in ns.
const uint32_t D_QKV = 600000, D_ATTN = 500000, D_PROJ = 200000, D_FC1 = 800000, D_FC2 = 800000;
const uint32_t D_EMB = 100000, D_LOSS = 300000, D_OPT = 5000000;
const uint32_t D_TP_AR = 150000, D_DP_AR = 2000000, D_MP_AR = 50000, D_EMB_AR = 1000000;

Program build_program(const Cfg& c, int s) {
  Program p;
  const int PP = c.pp, M = c.m, L = c.ls;
  const bool has_tp = c.tp > 1;
  auto fwd = [&](int mb) {
    if (s == 0) add_compute(p, 0, C_EMB, D_EMB, mb, 0);
    for (int l = 0; l < L; ++l) {
      add_compute(p, l, C_QKV, D_QKV, mb, 0);
      add_compute(p, l, C_ATTN, D_ATTN, mb, 0);
      add_compute(p, l, C_PROJ, D_PROJ, mb, 0);
      if (has_tp) add_coll(p, R_TP, O_TP_AR, D_TP_AR, mb, 0);
      add_compute(p, l, C_FC1, D_FC1, mb, 0);
      add_compute(p, l, C_FC2, D_FC2, mb, 0);
      if (has_tp) add_coll(p, R_TP, O_TP_AR, D_TP_AR, mb, 0);
    }
    if (s == PP - 1) add_compute(p, 0, C_LOSS, D_LOSS, mb, 0);
  };
  auto bwd = [&](int mb) {
    if (s == PP - 1) add_compute(p, 0, C_LOSS_B, D_LOSS, mb, 1);
    for (int l = L - 1; l >= 0; --l) {
      add_compute(p, l, C_FC2_B, 2 * D_FC2, mb, 1);
      add_compute(p, l, C_FC1_B, 2 * D_FC1, mb, 1);
      if (has_tp) add_coll(p, R_TP, O_TP_AR, D_TP_AR, mb, 1);
      add_compute(p, l, C_PROJ_B, 2 * D_PROJ, mb, 1);
      add_compute(p, l, C_ATTN_B, 2 * D_ATTN, mb, 1);
      add_compute(p, l, C_QKV_B, 2 * D_QKV, mb, 1);
      if (has_tp) add_coll(p, R_TP, O_TP_AR, D_TP_AR, mb, 1);
    }
    if (s == 0) add_compute(p, 0, C_EMB_B, 2 * D_EMB, mb, 1);
  };
  const bool first = (s == 0), last = (s == PP - 1);
  auto SEND = [](int dir, int mb, int bwdf, int warm) { return P2POp{1, (int8_t)dir, (uint8_t)warm, 0, META(mb, 0, bwdf, warm)}; };
  auto RECV = [](int dir, int mb, int bwdf) { return P2POp{0, (int8_t)dir, 0, 0, META(mb, 0, bwdf, 0)}; };

  // Megatron non-interleaved 1F1B (forward_backward_pipelining_without_interleaving).
  int num_warmup = std::min(PP - s - 1, M);
  int num_remaining = M - num_warmup;
  int fmb = 0, bmb = 0;
  for (int i = 0; i < num_warmup; ++i) {
    if (!first) add_p2p(p, {RECV(-1, fmb, 0)});
    fwd(fmb);
    // forward sends before the sender's first backward are warm-up
    if (!last) add_p2p(p, {SEND(+1, fmb, 0, 1)});
    ++fmb;
  }
  if (num_remaining > 0 && !first) add_p2p(p, {RECV(-1, fmb, 0)});
  for (int i = 0; i < num_remaining; ++i) {
    bool last_it = (i == num_remaining - 1);
    fwd(fmb);
    // first steady-state send still precedes this rank's first backward -> warm-up
    if (!last) add_p2p(p, {SEND(+1, fmb, 0, i == 0 ? 1 : 0), RECV(+1, bmb, 1)});
    ++fmb;
    bwd(bmb);
    if (last_it) {
      if (!first) add_p2p(p, {SEND(-1, bmb, 1, 0)});
    } else {
      if (!first) add_p2p(p, {SEND(-1, bmb, 1, 0), RECV(-1, fmb, 0)});
    }
    ++bmb;
  }
  for (int i = 0; i < num_warmup; ++i) {
    if (!last) add_p2p(p, {RECV(+1, bmb, 1)});
    bwd(bmb);
    if (!first) add_p2p(p, {SEND(-1, bmb, 1, 0)});
    ++bmb;
  }
  // iteration end: DP grad all-reduces (one bucket per layer), embedding AR, MP grad-norm AR, optimizer
  if (c.dp > 1)
    for (int l = 0; l < L; ++l) add_coll(p, R_DP, O_DP_AR, D_DP_AR, 0, 1);
  if (PP > 1 && (first || last)) add_coll(p, R_EMB, O_EMB_AR, D_EMB_AR, 0, 1);
  if (c.tp * c.pp > 1) add_coll(p, R_MP, O_MP_AR, D_MP_AR, 0, 1);
  add_compute(p, 0, C_OPT, D_OPT, 0, 1, /*iter_end=*/true);
  return p;
}

struct Topo {
  int tp, pp, dp, W;
  uint32_t nTP, nDP, nMP, nEMB, n_comms;
  int rank(int t, int d, int s) const { return t + tp * (d + dp * s); }
  int tp_of(int r) const { return r % tp; }
  int dp_of(int r) const { return (r / tp) % dp; }
  int pp_of(int r) const { return r / (tp * dp); }
  uint32_t comm_of(int r, int role) const {
    int t = tp_of(r), d = dp_of(r), s = pp_of(r);
    switch (role) {
      case R_TP: return (uint32_t)(s * dp + d);
      case R_DP: return nTP + (uint32_t)(s * tp + t);
      case R_MP: return nTP + nDP + (uint32_t)d;
      default:   return nTP + nDP + nMP + (uint32_t)(d * tp + t);
    }
  }
  void members(uint32_t c, std::vector<int>& out) const {
    out.clear();
    if (c < nTP) { int s = c / dp, d = c % dp; for (int t = 0; t < tp; ++t) out.push_back(rank(t, d, s)); return; }
    c -= nTP;
    if (c < nDP) { int s = c / tp, t = c % tp; for (int d = 0; d < dp; ++d) out.push_back(rank(t, d, s)); return; }
    c -= nDP;
    if (c < nMP) { int d = c; for (int s = 0; s < pp; ++s) for (int t = 0; t < tp; ++t) out.push_back(rank(t, d, s)); std::sort(out.begin(), out.end()); return; }
    c -= nMP;
    { int d = c / tp, t = c % tp; out.push_back(rank(t, d, 0)); out.push_back(rank(t, d, pp - 1)); }
  }
};

Topo make_topo(const Cfg& c) {
  Topo t; t.tp = c.tp; t.pp = c.pp; t.dp = c.dp; t.W = c.tp * c.pp * c.dp;
  t.nTP = c.tp > 1 ? (uint32_t)(c.dp * c.pp) : 0;
  t.nDP = c.dp > 1 ? (uint32_t)(c.tp * c.pp) : 0;
  t.nMP = c.tp * c.pp > 1 ? (uint32_t)c.dp : 0;
  t.nEMB = c.pp > 1 ? (uint32_t)(c.tp * c.dp) : 0;
  t.n_comms = t.nTP + t.nDP + t.nMP + t.nEMB;
  return t;
}

const int64_t LINK_LAT_NS = 20000;      // 20 us
const double LINK_BYTES_PER_NS = 25.0;  // 25 GB/s

// One iteration of the DES; writes events of iteration `it` for every rank.
struct IterSim {
  const Cfg& c; const Topo& T; const std::vector<Program>& progs;
  const uint64_t* rank_off; const std::vector<uint32_t>& comm_size;
  // outputs
  int64_t* start; uint32_t* dur; uint16_t* kind_op; uint16_t* meta; uint32_t* comm; uint32_t* payload;
  uint64_t* gt_inst; int64_t* makespan_out;
  // state
  std::vector<int64_t> t;          // per rank local (iteration-relative) time
  std::vector<uint32_t> pc;        // per rank op index
  std::vector<int64_t> arrive;     // per rank arrival time at a blocking op
  std::vector<uint32_t> coll_k, coll_n;   // per comm: next instance, arrivals so far
  std::vector<int64_t> coll_max;
  std::vector<std::vector<int>> comm_members;
  // P2P channel per (src, dir): sends from src to src+dir*stage_stride
  struct Post { int64_t time; int rank; uint32_t ev; };
  std::vector<std::vector<Post>> chan_send, chan_recv;  // index: src*2 + (dir>0)
  std::vector<uint32_t> chan_done;
  std::vector<int> pending;        // per rank pending p2p ops
  std::vector<int64_t> group_end;  // per rank
  std::vector<int> ready;
  uint64_t inst_counter = 0;
  uint32_t payload_bytes;
  int it;

  IterSim(const Cfg& c_, const Topo& T_, const std::vector<Program>& p_, const uint64_t* ro,
          const std::vector<uint32_t>& cs, const std::vector<std::vector<int>>& cm)
      : c(c_), T(T_), progs(p_), rank_off(ro), comm_size(cs), comm_members(cm) {
    t.resize(T.W); pc.resize(T.W); arrive.resize(T.W);
    coll_k.resize(T.n_comms); coll_n.resize(T.n_comms); coll_max.resize(T.n_comms);
    chan_send.resize((size_t)T.W * 2); chan_recv.resize((size_t)T.W * 2); chan_done.resize((size_t)T.W * 2);
    pending.resize(T.W); group_end.resize(T.W);
    int64_t pb = 2048LL * c.hidden * 2 / c.tp;
    payload_bytes = (uint32_t)std::min<int64_t>(pb, 0xFFFFFFFFll);
  }

  uint64_t ev_index(int r, uint32_t local) const {
    return rank_off[r] + (uint64_t)(it - c.it_begin) * progs[T.pp_of(r)].n_events + local;
  }

  double throttle_factor(int r, uint64_t opidx) const {
    double f = 1.0;
    for (auto& fl : c.faults)
      if (fl.type == 1 && fl.a == r && it >= fl.it0 && it < fl.it1) {
        if (fl.prob >= 1.0 || u01(rng4(c.seed ^ 0x7777, (uint64_t)it, (uint64_t)r, opidx)) < fl.prob) f *= fl.factor;
      }
    return f;
  }
  int64_t transfer_ns(int src, int dst, uint64_t k) const {
    double bw = LINK_BYTES_PER_NS, mult = 1.0;
    for (auto& fl : c.faults) {
      if (fl.a != src || fl.b != dst || it < fl.it0 || it >= fl.it1) continue;
      if (fl.type == 3) bw *= fl.factor;
      if (fl.type == 2) mult *= 1.0 + (-std::log(1.0 - u01(rng4(c.seed ^ 0x5151, (uint64_t)it, (uint64_t)src * 65536u + dst, k))));
    }
    double jit = 1.0 + c.jitter * (2.0 * u01(rng4(c.seed ^ 0x3333, (uint64_t)it, (uint64_t)src * 65536u + dst, k)) - 1.0);
    double x = ((double)LINK_LAT_NS + (double)payload_bytes / bw) * mult * jit;
    return (int64_t)std::llround(x);
  }

  void emit(uint64_t e, int64_t st, int64_t d, uint16_t ko, uint16_t me, uint32_t cm, uint32_t pl, uint64_t gi) {
    if (start) start[e] = st;
    dur[e] = (uint32_t)d; kind_op[e] = ko; meta[e] = me; comm[e] = cm; payload[e] = pl;
    if (gt_inst) gt_inst[e] = gi;
  }

  void complete_pair(int ch, uint32_t idx) {
    Post& s = chan_send[ch][idx];
    Post& r = chan_recv[ch][idx];
    int64_t E = std::max(s.time, r.time) + transfer_ns(s.rank, r.rank, idx);
    uint64_t gi = ((uint64_t)it << 40) | (inst_counter++);
    // SEND event on s.rank, RECV on r.rank
    uint64_t es = ev_index(s.rank, s.ev), er = ev_index(r.rank, r.ev);
    dur[es] = (uint32_t)(E - s.time); dur[er] = (uint32_t)(E - r.time);
    if (gt_inst) { gt_inst[es] = gi; gt_inst[er] = gi; }
    for (int who : {s.rank, r.rank}) {
      group_end[who] = std::max(group_end[who], E);
      if (--pending[who] == 0) { t[who] = group_end[who]; pc[who]++; ready.push_back(who); }
    }
  }

  void run(int iteration) {
    it = iteration;
    inst_counter = 0;
    std::fill(t.begin(), t.end(), 0); std::fill(pc.begin(), pc.end(), 0);
    std::fill(coll_k.begin(), coll_k.end(), 0); std::fill(coll_n.begin(), coll_n.end(), 0);
    std::fill(coll_max.begin(), coll_max.end(), INT64_MIN);
    for (auto& v : chan_send) v.clear();
    for (auto& v : chan_recv) v.clear();
    std::fill(chan_done.begin(), chan_done.end(), 0);
    std::vector<uint32_t> evcur(T.W, 0);
    ready.clear();
    for (int r = T.W - 1; r >= 0; --r) ready.push_back(r);
    while (!ready.empty()) {
      int r = ready.back(); ready.pop_back();
      const Program& P = progs[T.pp_of(r)];
      while (pc[r] < P.ops.size()) {
        const ProgOp& o = P.ops[pc[r]];
        uint32_t local = evcur[r];
        if (o.type == OT_COMPUTE) {
          uint64_t key = (uint64_t)local;
          double jit = 1.0 + c.jitter * (2.0 * u01(rng4(c.seed, (uint64_t)it, (uint64_t)r, key)) - 1.0);
          int64_t d = (int64_t)std::llround((double)o.base_dur * jit * throttle_factor(r, key));
          emit(ev_index(r, local), t[r], d, o.kind_op, o.meta, 0, 0, UINT64_MAX);
          t[r] += d; evcur[r]++; pc[r]++;
          continue;
        }
        if (o.type == OT_COLL) {
          uint32_t cid = T.comm_of(r, o.role);
          uint64_t e = ev_index(r, local);
          emit(e, t[r], 0, o.kind_op, o.meta, cid, 0, 0);
          arrive[r] = t[r];
          evcur[r]++;
          coll_max[cid] = std::max(coll_max[cid], t[r]);
          if (++coll_n[cid] == comm_size[cid]) {
            uint32_t k = coll_k[cid]++;
            double jit = 1.0 + c.jitter * (2.0 * u01(rng4(c.seed ^ 0x9999, (uint64_t)it, (uint64_t)cid, k)) - 1.0);
            int64_t E = coll_max[cid] + (int64_t)std::llround((double)o.base_dur * jit);
            uint64_t gi = ((uint64_t)it << 40) | (inst_counter++);
            for (int m : comm_members[cid]) {
              uint64_t em = ev_index(m, evcur[m] - 1);
              dur[em] = (uint32_t)(E - arrive[m]);
              if (gt_inst) gt_inst[em] = gi;
              t[m] = E; pc[m]++;
              if (m != r) ready.push_back(m);
            }
            coll_n[cid] = 0; coll_max[cid] = INT64_MIN;
            continue;  // r itself continues
          }
          break;  // blocked
        }
        // P2P group: post all ops, block until all complete
        pending[r] = o.n_p2p; group_end[r] = t[r];
        int my_stage = T.pp_of(r);
        std::vector<std::pair<int, uint32_t>> to_check;
        for (int q = 0; q < o.n_p2p; ++q) {
          const P2POp& x = o.p2p[q];
          int peer = T.rank(T.tp_of(r), T.dp_of(r), my_stage + x.dir);
          uint64_t e = ev_index(r, local + q);
          uint16_t ko = KO(x.is_send ? K_SEND : K_RECV, (uint16_t)((x.meta >> 13) & 1 ? O_P2P_GRAD : O_P2P_ACT));
          emit(e, t[r], 0, ko, x.meta, (uint32_t)peer, payload_bytes, 0);
          int src = x.is_send ? r : peer;
          int dir = x.is_send ? x.dir : -x.dir;  // direction from src to dst
          int ch = src * 2 + (dir > 0 ? 1 : 0);
          auto& vec = x.is_send ? chan_send[ch] : chan_recv[ch];
          vec.push_back(Post{t[r], r, local + q});
          to_check.push_back({ch, (uint32_t)vec.size() - 1});
        }
        evcur[r] += o.n_p2p;
        bool resumed = false;
        for (auto& pr : to_check) {
          int ch = pr.first; uint32_t idx = pr.second;
          if (idx < chan_send[ch].size() && idx < chan_recv[ch].size()) {
            bool was_pending = pending[r] > 0;
            complete_pair(ch, idx);
            if (was_pending && pending[r] == 0) resumed = true;
          }
        }
        if (resumed) {
          // complete_pair pushed r onto ready; pop it to continue inline
          for (size_t q = ready.size(); q-- > 0;) if (ready[q] == r) { ready.erase(ready.begin() + q); break; }
          continue;
        }
        break;
      }
    }
    int64_t ms = 0;
    for (int r = 0; r < T.W; ++r) {
      if (pc[r] != progs[T.pp_of(r)].ops.size()) { *makespan_out = -1; return; }  // deadlock
      ms = std::max(ms, t[r]);
    }
    *makespan_out = ms;
  }
};


}  // namespace


namespace {
Cfg to_cfg(const gen_config_c* g) {
  Cfg c;
  c.tp = g->tp; c.pp = g->pp; c.dp = g->dp; c.ls = g->layers_per_stage; c.m = g->microbatches;
  c.iters = g->iterations; c.seed = g->seed; c.hidden = g->hidden; c.jitter = g->jitter;
  c.skew = g->clock_skew; c.threads = g->n_threads;
  c.it_begin = g->it_begin; c.it_end = g->it_end ? g->it_end : g->iterations;
  for (int i = 0; i < g->n_faults; ++i) {
    const gen_fault_c& f = g->faults[i];
    c.faults.push_back(Fault{f.type, f.a, f.b, f.it0, f.it1, f.factor, f.prob});
  }
  return c;
}
}  // namespace

extern "C" {

// Per-rank event counts -> rank_offsets[W+1]; returns total events (or -1).
int64_t gen_count(const gen_config_c* g, uint64_t* rank_offsets) {
  Cfg c = to_cfg(g);
  if (c.tp < 1 || c.pp < 1 || c.dp < 1 || c.m < 1 || c.iters < 0 || c.ls < 1) return -1;
  if (c.it_begin < 0 || c.it_end < c.it_begin || c.it_end > c.iters) return -1;
  Topo T = make_topo(c);
  std::vector<uint32_t> per_stage(c.pp);
  for (int s = 0; s < c.pp; ++s) per_stage[s] = build_program(c, s).n_events;
  uint64_t off = 0;
  for (int r = 0; r < T.W; ++r) { rank_offsets[r] = off; off += (uint64_t)per_stage[T.pp_of(r)] * (c.it_end - c.it_begin); }
  rank_offsets[T.W] = off;
  return (int64_t)off;
}

// Comm table: returns n_comms; fills offsets[n_comms+1] and members (if non-null).
int64_t gen_comm_table(const gen_config_c* g, uint64_t* offsets, uint32_t* members) {
  Cfg c = to_cfg(g);
  Topo T = make_topo(c);
  std::vector<int> mem;
  uint64_t off = 0;
  for (uint32_t cid = 0; cid < T.n_comms; ++cid) {
    T.members(cid, mem);
    if (offsets) offsets[cid] = off;
    if (members) for (size_t i = 0; i < mem.size(); ++i) members[off + i] = (uint32_t)mem[i];
    off += mem.size();
  }
  if (offsets) offsets[T.n_comms] = off;
  return (int64_t)T.n_comms;
}

// Fill the event columns. Returns 0 on success, -1 deadlock, -2 bad config.
int gen_fill(const gen_config_c* g, const uint64_t* rank_offsets, int64_t* start_ns, uint32_t* dur,
             uint16_t* kind_op, uint16_t* meta, uint32_t* comm, uint32_t* payload,
             uint64_t* gt_inst, int64_t* gt_true_start) {
  Cfg c = to_cfg(g);
  if (c.tp < 1 || c.pp < 1 || c.dp < 1) return -2;
  const bool ranged = c.it_begin != 0 || c.it_end != c.iters;
  if (ranged && (start_ns || gt_inst || gt_true_start)) return -2;  // a range carries durations only
  if (c.it_begin < 0 || c.it_end < c.it_begin || c.it_end > c.iters) return -2;
  Topo T = make_topo(c);
  std::vector<Program> progs;
  for (int s = 0; s < c.pp; ++s) progs.push_back(build_program(c, s));
  std::vector<uint32_t> csize(T.n_comms);
  std::vector<std::vector<int>> cmem(T.n_comms);
  for (uint32_t cid = 0; cid < T.n_comms; ++cid) { T.members(cid, cmem[cid]); csize[cid] = (uint32_t)cmem[cid].size(); }
  std::vector<int64_t> makespan(c.iters, 0);
  int nth = c.threads > 0 ? c.threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nth = std::max(1, std::min(nth, std::max(1, c.it_end - c.it_begin)));
  std::atomic<int> next{c.it_begin};
  std::atomic<int> fail{0};
  auto worker = [&]() {
    IterSim sim(c, T, progs, rank_offsets, csize, cmem);
    sim.start = start_ns; sim.dur = dur; sim.kind_op = kind_op; sim.meta = meta; sim.comm = comm;
    sim.payload = payload; sim.gt_inst = gt_inst;
    for (;;) {
      int it = next.fetch_add(1);
      if (it >= c.it_end) break;
      sim.makespan_out = &makespan[it];
      sim.run(it);
      if (makespan[it] < 0) fail = 1;
    }
  };
  std::vector<std::thread> th;
  for (int i = 0; i < nth; ++i) th.emplace_back(worker);
  for (auto& x : th) x.join();
  if (fail) return -1;
  if (!start_ns) return 0;  // start times not requested (the analysis never reads them)
  // iteration start times: global barrier between iterations (+ 1 us gap)
  std::vector<int64_t> T0(c.iters + 1, 0);
  for (int i = 0; i < c.iters; ++i) T0[i + 1] = T0[i] + makespan[i] + 1000;
  std::vector<int64_t> off(T.W, 0);
  std::vector<double> drift(T.W, 0.0);
  if (c.skew)
    for (int r = 0; r < T.W; ++r) {
      off[r] = (int64_t)std::llround((2.0 * u01(rng4(c.seed ^ 0xC10C, 0, (uint64_t)r, 0)) - 1.0) * 2e6);
      drift[r] = (2.0 * u01(rng4(c.seed ^ 0xD21F, 0, (uint64_t)r, 0)) - 1.0) * 10e-6;
    }
  next = 0;
  auto fixer = [&]() {
    for (;;) {
      int r = next.fetch_add(1);
      if (r >= T.W) break;
      uint32_t ne = progs[T.pp_of(r)].n_events;
      for (int it = 0; it < c.iters; ++it) {
        uint64_t b = rank_offsets[r] + (uint64_t)it * ne;
        for (uint32_t q = 0; q < ne; ++q) {
          int64_t tru = start_ns[b + q] + T0[it];
          if (gt_true_start) gt_true_start[b + q] = tru;
          start_ns[b + q] = tru + off[r] + (int64_t)std::llround(drift[r] * (double)tru);
        }
      }
    }
  };
  th.clear();
  for (int i = 0; i < nth; ++i) th.emplace_back(fixer);
  for (auto& x : th) x.join();
  return 0;
}


// Per-rank Chrome-trace JSON documents of given event columns (the clean form of
// tracegen/chrome.py rank_documents(messy=False), byte for byte). Pass 1 (out == NULL): fills
// doc_off[W+1] and returns the total size; pass 2: writes the documents. Test infrastructure.
static void chrome_rank(std::string& o, uint32_t r, const uint64_t* ro, const int64_t* start, const uint32_t* dur,
                        const uint16_t* kind_op, const uint16_t* meta, const uint32_t* comm, const uint32_t* payload,
                        const uint64_t* coff, const uint32_t* cmem) {
  static const char* names[7] = {"compute", "all_reduce", "all_gather", "reduce_scatter", "broadcast", "send", "recv"};
  char tmp[64];
  auto us = [&](int64_t ns) {
    const bool neg = ns < 0;
    const uint64_t a = neg ? 0ull - (uint64_t)ns : (uint64_t)ns;
    if (a % 1000 == 0) snprintf(tmp, sizeof tmp, "%s%llu", neg ? "-" : "", (unsigned long long)(a / 1000));
    else snprintf(tmp, sizeof tmp, "%s%llu.%03llu", neg ? "-" : "", (unsigned long long)(a / 1000), (unsigned long long)(a % 1000));
    o += tmp;
  };
  auto num = [&](uint64_t v) { snprintf(tmp, sizeof tmp, "%llu", (unsigned long long)v); o += tmp; };
  o += "{\"traceEvents\":[";
  for (uint64_t i = ro[r]; i < ro[r + 1]; ++i) {
    if (i > ro[r]) o += ',';
    const uint32_t ko = kind_op[i], m = meta[i], kind = ko & 7u, iend = (ko >> 3) & 1u, op = ko >> 4;
    o += "{\"name\":\""; o += names[kind]; o += "\",\"cat\":\""; o += names[kind]; o += "\",\"ph\":\"X\",\"ts\":";
    us(start[i]);
    o += ",\"dur\":"; us((int64_t)dur[i]);
    o += ",\"pid\":"; num(r);
    o += kind == 0 ? ",\"tid\":0,\"args\":{" : ",\"tid\":1,\"args\":{";
    bool first = true;
    auto key = [&](const char* k) { if (!first) o += ','; first = false; o += '"'; o += k; o += "\":"; };
    if (op) { key("op"); num(op); }
    if (iend) { key("iter_end"); num(iend); }
    if (m & 1023u) { key("mb"); num(m & 1023u); }
    if ((m >> 10) & 7u) { key("chunk"); num((m >> 10) & 7u); }
    if ((m >> 13) & 1u) { key("bwd"); num(1); }
    if ((m >> 14) & 1u) { key("warmup"); num(1); }
    if (kind >= 1 && kind <= 4) {
      key("group");
      o += '[';
      for (uint64_t q = coff[comm[i]]; q < coff[comm[i] + 1]; ++q) { if (q > coff[comm[i]]) o += ','; num(cmem[q]); }
      o += ']';
    } else if (kind >= 5) {
      key("peer"); num(comm[i]);
    }
    if (payload[i]) { key("bytes"); num(payload[i]); }
    o += "}}";
  }
  o += "]}";
}

int64_t gen_chrome(uint32_t W, const uint64_t* ro, const int64_t* start, const uint32_t* dur, const uint16_t* kind_op,
                   const uint16_t* meta, const uint32_t* comm, const uint32_t* payload, const uint64_t* coff,
                   const uint32_t* cmem, uint8_t* out, uint64_t* doc_off, int n_threads) {
  if (n_threads <= 0) n_threads = (int)std::max(1u, std::thread::hardware_concurrency());
  n_threads = (int)std::min<uint32_t>((uint32_t)n_threads, std::max<uint32_t>(W, 1));
  std::vector<uint64_t> sz(W, 0);
  std::vector<std::thread> th;
  for (int t = 0; t < n_threads; ++t)
    th.emplace_back([&, t] {
      std::string o;
      for (uint32_t r = t; r < W; r += n_threads) {
        o.clear();
        chrome_rank(o, r, ro, start, dur, kind_op, meta, comm, payload, coff, cmem);
        sz[r] = o.size();
        if (out) memcpy(out + doc_off[r], o.data(), o.size());
      }
    });
  for (auto& x : th) x.join();
  if (!out) {
    doc_off[0] = 0;
    for (uint32_t r = 0; r < W; ++r) doc_off[r + 1] = doc_off[r] + sz[r];
  }
  return (int64_t)doc_off[W];
}

}  // extern "C"
