// k_json.cu — NEXT-2: Chrome-trace JSON ingest on the device and the merged, annotated emit.
//
// Ingest (P:L117-118 per-rank JSON files; P:L112 tracers.scope metadata; P:L131 participant lists;
// DESIGN.md §10d readings J1-J11). Data-parallel plan:
//   J-a  k_j_words   per 64-byte word: unescaped-quote / open / close bit masks (64 B read per word), the
//                    word's escape transfer code; a scan of the codes gives each word's entry state and
//                    k_j_escfix flips the one quote it changes (no look-back over backslash runs)
//   J-b  xor-scan of the per-word quote parity -> in-string state at every word start (CUB scan)
//   J-c  k_j_struct  string-filtered structural masks + depth delta per word; sum-scan -> depth
//   J-d  k_j_docs1 / k_j_marks / k_j_docs2 / k_j_arrclose / k_j_docs3: roots, the traceEvents
//        array of every document (bracket depth + atomics), document-level checks
//   J-e  k_j_count / k_j_place: the '{' of every event-array element (word counts + scan)
//   J-f  k_j_parse   one thread per element: validating JSON parse of the object, schema checks,
//                    exact decimal -> ns conversion, participant-list hash
//   J-g  program order (stable radix sorts by ts then rank), communicator interning in order of
//        first use (sort by group hash, exact verification, sort segments by first use), gather
//        into the event columns; then the ordinary load (scan_load_events, device pointers).
// Emit (P:L119-125 merged by time, pid = rank; P:L133 related_sync_op; J12): stable sort of the
// events by timestamp, per-event text length, scan, per-event write.
#include "internal.cuh"

#include <cub/cub.cuh>

namespace ms {
namespace {

enum : uint32_t {
  F_TRACE_EVENTS = 1, F_EVENT, F_PH, F_TS, F_DUR, F_PID, F_CAT, F_ARGS, F_OP, F_ITER_END, F_MB, F_CHUNK, F_BWD,
  F_WARMUP, F_GROUP, F_PEER, F_BYTES
};
constexpr uint64_t NONE64 = ~0ull;
#ifndef MS_J_CACHE
#define MS_J_CACHE 0   // 1: 16-byte register-cached cursor in k_j_parse (measured slower: registers)
#endif
#ifndef MS_J_PREFETCH
#define MS_J_PREFETCH 0   // k_j_parse: L1 prefetch of this many lines after an element's first (timed below)
#endif
#ifndef MS_J_MINB
#define MS_J_MINB 8    // k_j_parse: <= 64 registers, 16 warps per SM (measured: 1 -> 5.6 ms, 8 -> 3.2 ms on C2x40)
#endif
constexpr uint32_t SKIPPED = 0xFFFFFFFFu;

struct JErr {
  unsigned long long syn;     // smallest byte offset of a syntax error (~0 none)
  unsigned long long sch;     // smallest (offset << 8 | field) of a schema error
  unsigned long long collide; // group-hash collision (0 none)
  unsigned long long n_el;    // event-array elements
};

struct DocInfo {
  unsigned long long root, root_close, arr_open, arr_close;
  unsigned int te_keys, is_obj;
};

struct JsonState {
  DevBuf buf, docs, dinfo, err;
  DevBuf qm, om, cm, par, carry, delta, dbase, wcnt, wpre, esc, lead, ein;
  DevBuf epos, edoc;
  DevBuf e_rank, e_ts, e_dur, e_ko, e_meta, e_cp, e_pay, e_gh, e_gpos, e_gn;
  DevBuf keys_a, keys_b, vals_a, vals_b, tmp, flags, sel, nsel;
  DevBuf seg, segstart, first_j, seg_ord, comm_of_seg, ccnt, coff, cmem;
  DevBuf c_start, c_dur, c_kind, c_meta, c_comm, c_pay, c_roff;
  // emit
  DevBuf o_rank, o_inst, o_key, o_key2, o_perm, o_perm2, o_len, o_off, out;
  uint64_t out_bytes = 0, out_gen = ~0ull;
  uint32_t out_flags = 0;
  bool out_valid = false;
};

JsonState& js(Ctx& c) {
  if (!c.json_state) c.json_state = new JsonState();
  return *static_cast<JsonState*>(c.json_state);
}

__device__ __forceinline__ bool is_ws(uint32_t x) { return x == ' ' || x == '\t' || x == '\n' || x == '\r'; }

__device__ __forceinline__ uint32_t doc_of(const uint64_t* docs, uint32_t n_docs, uint64_t p) {
  uint32_t lo = 0, hi = n_docs;  // largest d with docs[d] <= p
  while (hi - lo > 1) {
    const uint32_t m = (lo + hi) >> 1;
    if (docs[m] <= p) lo = m; else hi = m;
  }
  return lo;
}

__device__ __forceinline__ uint64_t prefix_xor(uint64_t x) {
  x ^= x << 1; x ^= x << 2; x ^= x << 4; x ^= x << 8; x ^= x << 16; x ^= x << 32;
  return x;
}

// ------------------------------------------------------------------------------------- J-a .. J-c
// Escapes cross word boundaries: whether the first byte of a word is escaped depends on the
// backslash run ending the previous bytes. Each word is classified assuming it is NOT entered
// escaped; the only byte whose meaning flips when it is entered escaped is the first byte after its
// leading backslash run (a quote there toggles). The entry state itself comes from a scan of
// per-word transfer codes (esc): a word holding a non-backslash byte leaves the state given by the
// parity of its trailing run (0 / 1), an all-backslash word (64, even) passes it through (2). O(n).
__global__ void __launch_bounds__(256) k_j_words(const uint8_t* __restrict__ b, uint64_t n, uint64_t nw, uint64_t* qm,
                                                 uint64_t* om, uint64_t* cm, uint8_t* esc, uint8_t* lead) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nw) return;
  const uint64_t p0 = w * 64;
  uint32_t run = 0;      // backslashes since the last other byte
  uint32_t ld = 0;       // 0x80 | position of the first non-backslash byte if it is a quote, else 0
  bool other = false;    // a non-backslash byte seen
  uint64_t q = 0, o = 0, cl = 0;
  const uint4* v = reinterpret_cast<const uint4*>(b + p0);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint4 x = __ldg(v + k);
    const uint32_t wd[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t ch = (wd[j >> 2] >> (8 * (j & 3))) & 0xFFu;
      const int bit = k * 16 + j;
      if (p0 + bit >= n) continue;
      if (ch == '\\') { ++run; continue; }
      if (!other && ch == '"') ld = 0x80u | (uint32_t)bit;
      other = true;
      if (ch == '"' && !(run & 1)) q |= 1ull << bit;
      if (ch == '{' || ch == '[') o |= 1ull << bit;
      if (ch == '}' || ch == ']') cl |= 1ull << bit;
      run = 0;
    }
  }
  qm[w] = q; om[w] = o; cm[w] = cl;
  esc[w] = other ? (uint8_t)(run & 1) : (uint8_t)2;
  lead[w] = (uint8_t)ld;
}

// escape-state composition for the scan: a later constant wins, identity passes the earlier state
struct EscOp {
  __device__ __forceinline__ uint8_t operator()(uint8_t a, uint8_t b) const { return b == 2 ? a : b; }
};

// entered escaped: the leading quote flips; then the quote parity of the word
__global__ void __launch_bounds__(256) k_j_escfix(uint64_t nw, uint64_t* qm, const uint8_t* ein, const uint8_t* lead,
                                                  uint8_t* par) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nw) return;
  uint64_t q = qm[w];
  const uint8_t ld = lead[w];
  if (ein[w] == 1 && (ld & 0x80u)) { q ^= 1ull << (ld & 63u); qm[w] = q; }
  par[w] = (uint8_t)(__popcll(q) & 1);
}

__device__ __forceinline__ uint64_t instr_mask(uint64_t q, uint8_t carry) {
  return prefix_xor(q) ^ (carry ? ~0ull : 0ull);  // bit i: inside a string after byte i (opening quote: 1)
}

__global__ void __launch_bounds__(256) k_j_struct(uint64_t nw, const uint64_t* qm, uint64_t* om, uint64_t* cm,
                                                  const uint8_t* carry, int* delta) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nw) return;
  const uint64_t in = instr_mask(qm[w], carry[w]);
  const uint64_t o = om[w] & ~in, cl = cm[w] & ~in;
  om[w] = o; cm[w] = cl;
  delta[w] = __popcll(o) - __popcll(cl);
}

struct JA {
  const uint8_t* b; uint64_t n; const uint64_t* docs; uint32_t n_docs; uint64_t nw;
  const uint64_t* qm; const uint64_t* om; const uint64_t* cm; const uint8_t* carry; const int* dbase;
  DocInfo* di; JErr* err; const uint32_t* wpre; uint32_t* wcnt; uint64_t* epos; uint32_t* edoc;
};

__device__ __forceinline__ int depth_at(const JA& a, uint64_t p) {  // depth before byte p
  const uint64_t w = p >> 6;
  const uint64_t m = (p & 63) ? ((1ull << (p & 63)) - 1) : 0ull;
  return a.dbase[w] + __popcll(a.om[w] & m) - __popcll(a.cm[w] & m);
}
__device__ __forceinline__ bool in_string_before(const JA& a, uint64_t p) {
  const uint64_t w = p >> 6;
  const uint64_t m = (p & 63) ? ((1ull << (p & 63)) - 1) : 0ull;
  return ((__popcll(a.qm[w] & m) & 1) ^ a.carry[w]) != 0;
}
__device__ __forceinline__ void syn(JErr* e, uint64_t p) { atomicMin(&e->syn, (unsigned long long)p); }
__device__ __forceinline__ void sch(JErr* e, uint64_t p, uint32_t f) { atomicMin(&e->sch, (unsigned long long)((p << 8) | f)); }

__global__ void k_j_docs1(JA a) {
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= a.n_docs) return;
  const uint64_t s = a.docs[d], e = a.docs[d + 1];
  DocInfo& I = a.di[d];
  I.root = I.root_close = I.arr_open = I.arr_close = NONE64;
  I.te_keys = 0; I.is_obj = 0;
  if (s < a.n && (in_string_before(a, s) || depth_at(a, s) != 0)) { syn(a.err, s); return; }
  uint64_t p = s;
  while (p < e && is_ws(a.b[p])) ++p;
  if (p >= e) { syn(a.err, p); return; }
  const uint8_t ch = a.b[p];
  if (ch != '{' && ch != '[') { syn(a.err, p); return; }
  I.root = p; I.is_obj = ch == '{';
  if (ch == '[') I.arr_open = p;
}

// root closes (depth 1 -> 0), stray closes (depth 0), "traceEvents": keys of object roots
__global__ void __launch_bounds__(256) k_j_marks(JA a) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= a.nw) return;
  const uint64_t cl = a.cm[w];
  const uint64_t qo = a.qm[w] & instr_mask(a.qm[w], a.carry[w]);  // opening quotes
  uint64_t cand = cl | qo;
  if (!cand) return;
  uint32_t d = doc_of(a.docs, a.n_docs, w * 64);
  while (cand) {
    const int bit = __ffsll((long long)cand) - 1;
    cand &= cand - 1;
    const uint64_t p = w * 64 + bit;
    while (d + 1 < a.n_docs && p >= a.docs[d + 1]) ++d;
    const int dep = depth_at(a, p);
    if ((cl >> bit) & 1) {
      if (dep <= 0) syn(a.err, p);
      else if (dep == 1) atomicMin(&a.di[d].root_close, (unsigned long long)p);
      continue;
    }
    if (dep != 1) continue;
    const uint64_t e = a.docs[d + 1];
    const char* key = "\"traceEvents\"";
    if (p + 13 > e) continue;
    bool ok = true;
    for (int k = 0; k < 13 && ok; ++k) ok = a.b[p + k] == (uint8_t)key[k];
    if (!ok) continue;
    uint64_t q = p + 13;
    while (q < e && is_ws(a.b[q])) ++q;
    if (q >= e || a.b[q] != ':') continue;
    atomicAdd(&a.di[d].te_keys, 1u);
    ++q;
    while (q < e && is_ws(a.b[q])) ++q;
    if (q < e && a.b[q] == '[') atomicMin(&a.di[d].arr_open, (unsigned long long)q);
  }
}

__global__ void k_j_docs2(JA a) {
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= a.n_docs) return;
  DocInfo& I = a.di[d];
  if (I.root == NONE64) return;
  const uint64_t e = a.docs[d + 1];
  if (I.root_close == NONE64 || I.root_close >= e) { syn(a.err, I.root); return; }
  for (uint64_t p = I.root_close + 1; p < e; ++p)
    if (!is_ws(a.b[p])) { syn(a.err, p); return; }
  if (I.is_obj && (I.te_keys != 1 || I.arr_open == NONE64)) { sch(a.err, I.root, F_TRACE_EVENTS); I.arr_open = NONE64; }
  if (!I.is_obj) I.arr_close = I.root_close;
}

__global__ void __launch_bounds__(256) k_j_arrclose(JA a) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= a.nw) return;
  uint64_t cand = a.cm[w];
  if (!cand) return;
  uint32_t d = doc_of(a.docs, a.n_docs, w * 64);
  while (cand) {
    const int bit = __ffsll((long long)cand) - 1;
    cand &= cand - 1;
    const uint64_t p = w * 64 + bit;
    while (d + 1 < a.n_docs && p >= a.docs[d + 1]) ++d;
    const DocInfo& I = a.di[d];
    if (!I.is_obj || I.arr_open == NONE64 || p <= I.arr_open) continue;
    if (depth_at(a, p) == 2) atomicMin(&a.di[d].arr_close, (unsigned long long)p);
  }
}

__device__ __forceinline__ uint64_t elem_mask(const JA& a, uint64_t w, uint32_t& d) {
  // '{' at depth (array depth + 1) inside the event array of their document
  uint64_t o = a.om[w], out = 0;
  if (!o) return 0;
  d = doc_of(a.docs, a.n_docs, w * 64);
  while (o) {
    const int bit = __ffsll((long long)o) - 1;
    o &= o - 1;
    const uint64_t p = w * 64 + bit;
    uint32_t dd = d;
    while (dd + 1 < a.n_docs && p >= a.docs[dd + 1]) ++dd;
    const DocInfo& I = a.di[dd];
    if (I.arr_open == NONE64 || I.arr_close == NONE64 || p <= I.arr_open || p >= I.arr_close) continue;
    if (a.b[p] != '{') continue;
    if (depth_at(a, p) == (I.is_obj ? 2 : 1)) out |= 1ull << bit;
  }
  return out;
}

__global__ void __launch_bounds__(256) k_j_count(JA a) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= a.nw) return;
  uint32_t d = 0;
  a.wcnt[w] = __popcll(elem_mask(a, w, d));
}

__global__ void __launch_bounds__(256) k_j_place(JA a) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= a.nw) return;
  uint32_t d = 0;
  uint64_t m = elem_mask(a, w, d);
  uint32_t i = a.wpre[w];
  while (m) {
    const int bit = __ffsll((long long)m) - 1;
    m &= m - 1;
    const uint64_t p = w * 64 + bit;
    while (d + 1 < a.n_docs && p >= a.docs[d + 1]) ++d;
    a.epos[i] = p; a.edoc[i] = d; ++i;
  }
}

// ------------------------------------------------------------------------------------- J-f parser
struct Cur {
  const uint8_t* b; uint64_t p, end, bad;
  uint64_t cb = ~0ull;   // 16-byte block cached in registers (the input buffer is padded and aligned)
  uint4 cv;
  __device__ __forceinline__ uint32_t c() {
    if (p >= end) return 0u;
#if MS_J_CACHE
    const uint64_t blk = p & ~15ull;
    if (blk != cb) { cb = blk; cv = __ldg(reinterpret_cast<const uint4*>(b + blk)); }
    const uint32_t q = (uint32_t)(p >> 2) & 3u;
    const uint32_t w = (q & 2u) ? ((q & 1u) ? cv.w : cv.z) : ((q & 1u) ? cv.y : cv.x);
    return (w >> (8u * ((uint32_t)p & 3u))) & 0xFFu;
#else
    return __ldg(b + p);
#endif
  }
  __device__ __forceinline__ void ws() { while (is_ws(c()) && p < end) ++p; }
  __device__ __forceinline__ bool fail() { if (bad == NONE64) bad = p; return false; }
};

// first 16 raw bytes of a key / string value, packed little-endian (keys and kind names fit)
constexpr uint64_t pk(const char* s, int off = 0) {
  uint64_t v = 0;
  for (int k = 0; k < 8 && s[off + k]; ++k) v |= (uint64_t)(uint8_t)s[off + k] << (8 * k);
  return v;
}
constexpr uint32_t slen(const char* s) { uint32_t n = 0; while (s[n]) ++n; return n; }
struct Str { uint64_t s; uint32_t len; uint64_t k0, k1; };
__device__ __forceinline__ bool is(const Str& x, const char* lit) {
  return x.len == slen(lit) && x.k0 == pk(lit) && x.k1 == (slen(lit) > 8 ? pk(lit, 8) : 0ull);
}

// JSON string at the cursor (validated: escapes, no control characters); raw content [s, s+len),
// its first 16 raw bytes packed into k0 / k1
__device__ bool j_string(Cur& u, Str& o) {
  if (u.c() != '"') return u.fail();
  ++u.p;
  o.s = u.p; o.k0 = 0; o.k1 = 0;
  while (true) {
    const uint32_t x = u.c();
    if (u.p >= u.end || x < 0x20) return u.fail();
    if (x == '"') break;
    const uint64_t n = u.p - o.s;
    if (n < 8) o.k0 |= (uint64_t)x << (8 * n);
    else if (n < 16) o.k1 |= (uint64_t)x << (8 * (n - 8));
    if (x == '\\') {
      ++u.p;
      const uint32_t y = u.c();
      if (y == 'u') {
        for (int k = 0; k < 4; ++k) {
          ++u.p;
          const uint32_t h = u.c();
          const bool hex = (h >= '0' && h <= '9') || (h >= 'a' && h <= 'f') || (h >= 'A' && h <= 'F');
          if (!hex) return u.fail();
        }
        ++u.p;
        continue;
      }
      if (!(y == '"' || y == '\\' || y == '/' || y == 'b' || y == 'f' || y == 'n' || y == 'r' || y == 't')) return u.fail();
      ++u.p;
      continue;
    }
    ++u.p;
  }
  o.len = (uint32_t)(u.p - o.s);
  ++u.p;
  return true;
}

struct Num {
  bool neg, ovf, has_frac, has_exp;
  uint64_t ip;          // integer part (valid if !ovf)
  uint32_t nfrac, frac3;
};

// JSON number grammar: -? (0 | [1-9][0-9]*) (. [0-9]+)? ([eE] [+-]? [0-9]+)?
__device__ bool j_number(Cur& u, Num& n) {
  n = Num{false, false, false, false, 0, 0, 0};
  if (u.c() == '-') { n.neg = true; ++u.p; }
  uint32_t x = u.c();
  if (x < '0' || x > '9') return u.fail();
  if (x == '0') {
    ++u.p;
  } else {
    while ((x = u.c()) >= '0' && x <= '9') {
      const uint64_t d = x - '0';
      if (n.ip > (~0ull - d) / 10) n.ovf = true; else n.ip = n.ip * 10 + d;
      ++u.p;
    }
  }
  if (u.c() == '.') {
    ++u.p;
    n.has_frac = true;
    if ((x = u.c()) < '0' || x > '9') return u.fail();
    while ((x = u.c()) >= '0' && x <= '9') {
      if (n.nfrac < 3) n.frac3 = n.frac3 * 10 + (x - '0');
      ++n.nfrac;
      ++u.p;
    }
  }
  x = u.c();
  if (x == 'e' || x == 'E') {
    ++u.p;
    n.has_exp = true;
    x = u.c();
    if (x == '+' || x == '-') { ++u.p; x = u.c(); }
    if (x < '0' || x > '9') return u.fail();
    while ((x = u.c()) >= '0' && x <= '9') ++u.p;
  }
  return true;
}

__device__ bool j_literal(Cur& u, const char* lit) {
  for (int k = 0; lit[k]; ++k) {
    if (u.c() != (uint8_t)lit[k]) return u.fail();
    ++u.p;
  }
  return true;
}

// validate and skip any JSON value (nesting <= 64 inside an event, reading J10)
__device__ bool j_skip(Cur& u) {
  uint64_t stk = 0;  // bit k: container at nesting k+1 is an object
  int dep = 0;
  bool want_key = false;
  while (true) {
    u.ws();
    if (want_key) {
      Str t;
      if (!j_string(u, t)) return false;
      u.ws();
      if (u.c() != ':') return u.fail();
      ++u.p;
      u.ws();
      want_key = false;
    }
    const uint32_t x = u.c();
    if (x == '{' || x == '[') {
      if (dep >= 64) return u.fail();
      const bool obj = x == '{';
      stk = obj ? (stk | (1ull << dep)) : (stk & ~(1ull << dep));
      ++dep;
      ++u.p;
      u.ws();
      if (u.c() == (obj ? '}' : ']')) { ++u.p; --dep; }
      else if (obj) { want_key = true; continue; }
      else continue;
    } else if (x == '"') {
      Str t;
      if (!j_string(u, t)) return false;
    } else if (x == '-' || (x >= '0' && x <= '9')) {
      Num n;
      if (!j_number(u, n)) return false;
    } else if (x == 't') { if (!j_literal(u, "true")) return false; }
    else if (x == 'f') { if (!j_literal(u, "false")) return false; }
    else if (x == 'n') { if (!j_literal(u, "null")) return false; }
    else return u.fail();
    // after a value: close containers / next element
    while (true) {
      if (dep == 0) return true;
      u.ws();
      const bool obj = (stk >> (dep - 1)) & 1;
      const uint32_t y = u.c();
      if (y == ',') { ++u.p; want_key = obj; break; }
      if (y == (obj ? '}' : ']')) { ++u.p; --dep; continue; }
      return u.fail();
    }
  }
}


// Elements of an event array that are not objects, from the cursor (just after '[' or after a
// ','): each must be a valid JSON value (else a syntax error) and is a schema error (SCAN_JF_EVENT)
// at its first byte; stops at the next object (parsed by its own thread) or at the array end.
__device__ void j_gap(Cur& u, uint64_t arr_close, bool after_comma, JErr* err) {
  while (true) {
    u.ws();
    const uint32_t x = u.c();
    if (x == '{') return;
    if (x == ']' && u.p == arr_close) {
      if (after_comma) syn(err, u.p);
      return;
    }
    const uint64_t v0 = u.p;
    if (!j_skip(u)) { syn(err, u.bad); return; }
    sch(err, v0, F_EVENT);
    u.ws();
    if (u.c() == ',') { ++u.p; after_comma = true; continue; }
    if (!(u.c() == ']' && u.p == arr_close)) syn(err, u.p);
    return;
  }
}

// per document (one thread): (1) an object root's members: keys, ':' and ',' and every member value
// are validated (the traceEvents array is skipped through its known close, its elements have their
// own parsers); (2) the elements before the first object of the event array (normally none)
__global__ void k_j_docs3(JA a) {
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= a.n_docs) return;
  const DocInfo& I = a.di[d];
  if (I.root != NONE64 && I.is_obj && I.root_close != NONE64) {
    Cur u{a.b, I.root + 1, I.root_close + 1, NONE64};
    u.ws();
    if (u.c() == '}' && u.p == I.root_close) {
      // empty root object (no traceEvents: reported by k_j_docs2)
    } else {
      while (true) {
        u.ws();
        Str k;
        if (!j_string(u, k)) { syn(a.err, u.bad); break; }
        u.ws();
        if (u.c() != ':') { syn(a.err, u.p); break; }
        ++u.p;
        u.ws();
        if (u.p == I.arr_open && I.arr_close != NONE64) u.p = I.arr_close + 1;  // the event array
        else if (!j_skip(u)) { syn(a.err, u.bad); break; }
        u.ws();
        if (u.c() == ',') { ++u.p; continue; }
        if (!(u.c() == '}' && u.p == I.root_close)) syn(a.err, u.p);
        break;
      }
    }
  }
  if (I.arr_open == NONE64 || I.arr_close == NONE64) return;
  Cur u{a.b, I.arr_open + 1, I.arr_close + 1, NONE64};
  j_gap(u, I.arr_close, false, a.err);
}

__constant__ char KNAME[7][16] = {"compute", "all_reduce", "all_gather", "reduce_scatter", "broadcast", "send", "recv"};

struct Ev {
  uint32_t pres, bad;
  bool ph_x;
  int64_t ts;
  uint32_t dur, pid, kind, op, iter_end, mb, chunk, bwd, warmup, peer, bytes, gn;
  uint64_t gh, gpos;
};

__device__ __forceinline__ void setf(Ev& v, uint32_t f, bool ok) {
  v.pres |= 1u << f;
  v.bad = ok ? (v.bad & ~(1u << f)) : (v.bad | (1u << f));
}

// ts / dur: microseconds with <= 3 decimals -> ns, exact, in [lo, hi] (J5)
__device__ bool usec_ns(const Num& n, bool is_ts, int64_t& out) {
  if (n.has_exp || n.nfrac > 3 || n.ovf) return false;
  uint32_t f = n.frac3;
  for (uint32_t k = n.nfrac; k < 3; ++k) f *= 10;
  if (n.ip > (~0ull - 999) / 1000) return false;
  const uint64_t m = n.ip * 1000 + f;
  if (is_ts) {
    if (n.neg) { if (m > (1ull << 63)) return false; out = (int64_t)(0ull - m); }
    else { if (m > (uint64_t)INT64_MAX) return false; out = (int64_t)m; }
  } else {
    if (n.neg && m != 0) return false;
    if (m > 0xFFFFFFFFull) return false;
    out = (int64_t)m;
  }
  return true;
}

__device__ bool int_in(const Num& n, uint64_t hi, uint32_t& out) {
  if (n.has_frac || n.has_exp || n.ovf) return false;
  if (n.neg && n.ip != 0) return false;
  if (n.ip > hi) return false;
  out = (uint32_t)n.ip;
  return true;
}

// value of an integer field: a number in [0, hi]; flags (hi == 1) also accept true / false
__device__ bool j_int_field(Cur& u, uint64_t hi, bool flag, uint32_t& out, bool& ok) {
  const uint32_t x = u.c();
  ok = false;
  if (x == '-' || (x >= '0' && x <= '9')) {
    Num n;
    if (!j_number(u, n)) return false;
    ok = int_in(n, hi, out);
    return true;
  }
  if (flag && (x == 't' || x == 'f')) {
    if (!j_literal(u, x == 't' ? "true" : "false")) return false;
    out = x == 't';
    ok = true;
    return true;
  }
  return j_skip(u);
}

// a repeated "args" key replaces the earlier one: back to defaults
__device__ void args_reset(Ev& v) {
  v.op = v.iter_end = v.mb = v.chunk = v.bwd = v.warmup = v.peer = v.bytes = v.gn = 0;
  v.gh = 0; v.gpos = NONE64;
  const uint32_t amask = (1u << F_OP) | (1u << F_ITER_END) | (1u << F_MB) | (1u << F_CHUNK) | (1u << F_BWD) |
                         (1u << F_WARMUP) | (1u << F_GROUP) | (1u << F_PEER) | (1u << F_BYTES);
  v.pres &= ~amask; v.bad &= ~amask;
}

__device__ bool j_args(Cur& u, Ev& v, uint32_t world) {
  args_reset(v);
  ++u.p;  // '{'
  u.ws();
  if (u.c() == '}') { ++u.p; return true; }
  while (true) {
    u.ws();
    Str k;
    if (!j_string(u, k)) return false;
    u.ws();
    if (u.c() != ':') return u.fail();
    ++u.p;
    u.ws();
    uint32_t f = 0;
    uint64_t hi = 0;
    if (is(k, "op")) { f = F_OP; hi = 4095; }
    else if (is(k, "iter_end")) { f = F_ITER_END; hi = 1; }
    else if (is(k, "mb")) { f = F_MB; hi = 1023; }
    else if (is(k, "chunk")) { f = F_CHUNK; hi = 7; }
    else if (is(k, "bwd")) { f = F_BWD; hi = 1; }
    else if (is(k, "warmup")) { f = F_WARMUP; hi = 1; }
    else if (is(k, "peer")) { f = F_PEER; hi = (uint64_t)world - 1; }
    else if (is(k, "bytes")) { f = F_BYTES; hi = 0xFFFFFFFFull; }
    if (f) {
      bool ok = false;
      uint32_t val = 0;
      if (!j_int_field(u, hi, f == F_ITER_END || f == F_BWD || f == F_WARMUP, val, ok)) return false;
      setf(v, f, ok);
      switch (f) {
        case F_OP: v.op = val; break;
        case F_ITER_END: v.iter_end = val; break;
        case F_MB: v.mb = val; break;
        case F_CHUNK: v.chunk = val; break;
        case F_BWD: v.bwd = val; break;
        case F_WARMUP: v.warmup = val; break;
        case F_PEER: v.peer = val; break;
        default: v.bytes = val; break;
      }
    } else if (is(k, "group")) {
      if (u.c() != '[') {
        if (!j_skip(u)) return false;
        setf(v, F_GROUP, false);
      } else {
        v.gpos = u.p;
        ++u.p;
        uint64_t h = 1469598103934665603ull;
        uint32_t cnt = 0, prev = 0;
        bool gok = true;
        u.ws();
        if (u.c() == ']') { ++u.p; gok = false; }
        else {
          while (true) {
            u.ws();
            const uint32_t x = u.c();
            if (x == '-' || (x >= '0' && x <= '9')) {
              Num n;
              if (!j_number(u, n)) return false;
              uint32_t m = 0;
              if (!int_in(n, (uint64_t)world - 1, m) || (cnt && m <= prev)) gok = false;
              prev = m;
              h = (h ^ m) * 1099511628211ull;
              ++cnt;
            } else {
              if (!j_skip(u)) return false;
              gok = false;
            }
            u.ws();
            if (u.c() == ',') { ++u.p; continue; }
            if (u.c() == ']') { ++u.p; break; }
            return u.fail();
          }
        }
        setf(v, F_GROUP, gok);
        v.gh = h; v.gn = cnt;
      }
    } else {
      if (!j_skip(u)) return false;
    }
    u.ws();
    if (u.c() == ',') { ++u.p; continue; }
    if (u.c() == '}') { ++u.p; return true; }
    return u.fail();
  }
}

struct PA {
  const uint8_t* b; const uint64_t* epos; const uint32_t* edoc; const DocInfo* di; uint64_t n_el; uint32_t world;
  JErr* err;
  uint32_t* rank; int64_t* ts; uint32_t* dur; uint16_t* ko; uint16_t* meta; uint32_t* cp; uint32_t* pay;
  uint64_t* gh; uint64_t* gpos; uint32_t* gn;
};

__global__ void __launch_bounds__(128, MS_J_MINB) k_j_parse(PA a) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n_el) return;
  const uint64_t p0 = a.epos[i];
  const DocInfo& I = a.di[a.edoc[i]];
#if MS_J_PREFETCH
  {  // the element's first lines (typical elements span 2-3): later misses overlap the first
    const uint64_t lim = I.arr_close + 1;
    for (uint32_t k = 1; k <= MS_J_PREFETCH; ++k)
      if (p0 + 128ull * k < lim) asm volatile("prefetch.global.L1 [%0];" ::"l"(a.b + p0 + 128ull * k));
  }
#endif
  Cur u{a.b, p0, I.arr_close + 1, NONE64};
  Ev v{};
  v.gpos = NONE64;
  bool ok = true;
  // the event object
  ++u.p;
  u.ws();
  if (u.c() == '}') ++u.p;
  else {
    while (ok) {
      u.ws();
      Str k;
      if (!j_string(u, k)) { ok = false; break; }
      u.ws();
      if (u.c() != ':') { ok = u.fail(); break; }
      ++u.p;
      u.ws();
      const uint32_t x = u.c();
      if (is(k, "ph")) {
        if (x == '"') {
          Str t;
          if (!j_string(u, t)) { ok = false; break; }
          setf(v, F_PH, true);
          v.ph_x = t.len == 1 && t.k0 == 'X';
        } else {
          if (!j_skip(u)) { ok = false; break; }
          setf(v, F_PH, false);
        }
      } else if (is(k, "ts") || is(k, "dur")) {
        const bool is_ts = k.len == 2;
        bool good = false;
        int64_t ns = 0;
        if (x == '-' || (x >= '0' && x <= '9')) {
          Num n;
          if (!j_number(u, n)) { ok = false; break; }
          good = usec_ns(n, is_ts, ns);
        } else if (!j_skip(u)) { ok = false; break; }
        setf(v, is_ts ? F_TS : F_DUR, good);
        if (is_ts) v.ts = ns; else v.dur = (uint32_t)ns;
      } else if (is(k, "pid")) {
        bool good;
        uint32_t val = 0;
        if (!j_int_field(u, (uint64_t)a.world - 1, false, val, good)) { ok = false; break; }
        setf(v, F_PID, good);
        v.pid = val;
      } else if (is(k, "cat")) {
        bool good = false;
        if (x == '"') {
          Str t;
          if (!j_string(u, t)) { ok = false; break; }
          const char* names[7] = {"compute", "all_reduce", "all_gather", "reduce_scatter", "broadcast", "send", "recv"};
#pragma unroll
          for (uint32_t q = 0; q < 7; ++q)
            if (is(t, names[q])) { good = true; v.kind = q; }
        } else if (!j_skip(u)) { ok = false; break; }
        setf(v, F_CAT, good);
      } else if (is(k, "args")) {
        if (x == '{') {
          if (!j_args(u, v, a.world)) { ok = false; break; }
          setf(v, F_ARGS, true);
        } else {
          if (!j_skip(u)) { ok = false; break; }
          args_reset(v);
          setf(v, F_ARGS, false);
        }
      } else {
        if (!j_skip(u)) { ok = false; break; }
      }
      u.ws();
      if (u.c() == ',') { ++u.p; continue; }
      if (u.c() == '}') { ++u.p; break; }
      ok = u.fail();
    }
  }
  if (ok) {  // separator after the element: ',' + next element (must be an object) or the array end
    u.ws();
    const uint32_t x = u.c();
    if (x == ',') {
      ++u.p;
      j_gap(u, I.arr_close, true, a.err);
    } else if (!(x == ']' && u.p == I.arr_close)) ok = u.fail();
  }
  if (!ok) {
    syn(a.err, u.bad == NONE64 ? p0 : u.bad);
    a.rank[i] = SKIPPED;
    return;
  }
  // schema (J6-J9, J11: first failing field in this order)
  uint32_t f = 0;
  const auto missing_or_bad = [&](uint32_t fl) { return !((v.pres >> fl) & 1) || ((v.bad >> fl) & 1); };
  const auto bad = [&](uint32_t fl) { return ((v.bad >> fl) & 1) != 0; };
  if (missing_or_bad(F_PH)) f = F_PH;
  else if (!v.ph_x) { a.rank[i] = SKIPPED; return; }
  else if (missing_or_bad(F_TS)) f = F_TS;
  else if (missing_or_bad(F_DUR)) f = F_DUR;
  else if (missing_or_bad(F_PID)) f = F_PID;
  else if (missing_or_bad(F_CAT)) f = F_CAT;
  else if (bad(F_ARGS)) f = F_ARGS;
  else if (bad(F_OP)) f = F_OP;
  else if (bad(F_ITER_END)) f = F_ITER_END;
  else if (bad(F_MB)) f = F_MB;
  else if (bad(F_CHUNK)) f = F_CHUNK;
  else if (bad(F_BWD)) f = F_BWD;
  else if (bad(F_WARMUP)) f = F_WARMUP;
  else if (v.kind >= 1 && v.kind <= 4 && missing_or_bad(F_GROUP)) f = F_GROUP;
  else if (v.kind >= 5 && missing_or_bad(F_PEER)) f = F_PEER;
  else if (bad(F_BYTES)) f = F_BYTES;
  if (f) { sch(a.err, p0, f); a.rank[i] = SKIPPED; return; }
  const bool coll = v.kind >= 1 && v.kind <= 4;
  a.rank[i] = v.pid;
  a.ts[i] = v.ts;
  a.dur[i] = v.dur;
  a.ko[i] = (uint16_t)(v.kind | (v.iter_end << 3) | (v.op << 4));
  a.meta[i] = (uint16_t)(v.mb | (v.chunk << 10) | (v.bwd << 13) | (v.warmup << 14));
  a.cp[i] = v.kind >= 5 ? v.peer : 0u;
  a.pay[i] = v.bytes;
  a.gh[i] = coll ? v.gh : 0ull;
  a.gpos[i] = coll ? v.gpos : NONE64;
  a.gn[i] = coll ? v.gn : 0u;
}

// ------------------------------------------------------------------------------------- J-g
__global__ void k_j_rankkeys(uint64_t n, const uint32_t* perm, const uint32_t* rank, uint32_t W, uint32_t* key) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint32_t r = rank[perm[j]];
  key[j] = r == SKIPPED ? W : r;
}

// rank offsets from the rank-sorted keys
__global__ void k_j_roff(uint64_t n, const uint32_t* key, uint32_t W, uint64_t* roff) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > W) return;
  uint64_t lo = 0, hi = n;  // first j with key[j] >= r
  while (lo < hi) {
    const uint64_t m = (lo + hi) >> 1;
    if (key[m] < r) lo = m + 1; else hi = m;
  }
  roff[r] = lo;
}

struct GA {
  uint64_t n; const uint32_t* perm;
  const int64_t* e_ts; const uint32_t* e_dur; const uint16_t* e_ko; const uint16_t* e_meta; const uint32_t* e_cp;
  const uint32_t* e_pay; const uint64_t* e_gh;
  int64_t* start; uint32_t* dur; uint16_t* kind; uint16_t* meta; uint32_t* comm; uint32_t* pay;
  uint8_t* is_coll; uint64_t* gkey;
};

__global__ void k_j_gather(GA a) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.n) return;
  const uint32_t i = a.perm[j];
  a.start[j] = a.e_ts[i]; a.dur[j] = a.e_dur[i]; a.kind[j] = a.e_ko[i]; a.meta[j] = a.e_meta[i];
  a.comm[j] = a.e_cp[i]; a.pay[j] = a.e_pay[i];
  const uint32_t k = a.e_ko[i] & 7u;
  a.is_coll[j] = k >= 1 && k <= 4;
  a.gkey[j] = a.e_gh[i];
}

__device__ uint32_t read_group(const uint8_t* b, uint64_t pos, uint32_t* out, uint32_t cap) {
  // a validated group array at pos ('['): integers separated by ',' and whitespace
  uint64_t p = pos + 1;
  uint32_t k = 0;
  while (true) {
    while (is_ws(b[p])) ++p;
    if (b[p] == ']') return k;
    uint32_t v = 0;
    if (b[p] == '-') ++p;
    while (b[p] >= '0' && b[p] <= '9') { v = v * 10 + (b[p] - '0'); ++p; }
    if (k < cap && out) out[k] = v;
    ++k;
    while (is_ws(b[p])) ++p;
    if (b[p] == ',') ++p;
  }
}

__device__ bool same_group(const uint8_t* b, uint64_t pa, uint64_t pb) {
  uint64_t p = pa + 1, q = pb + 1;
  while (true) {
    while (is_ws(b[p])) ++p;
    while (is_ws(b[q])) ++q;
    const bool ea = b[p] == ']', eb = b[q] == ']';
    if (ea || eb) return ea && eb;
    uint64_t x = 0, y = 0;
    if (b[p] == '-') ++p;
    if (b[q] == '-') ++q;
    while (b[p] >= '0' && b[p] <= '9') { x = x * 10 + (b[p] - '0'); ++p; }
    while (b[q] >= '0' && b[q] <= '9') { y = y * 10 + (b[q] - '0'); ++q; }
    if (x != y) return false;
    while (is_ws(b[p])) ++p;
    while (is_ws(b[q])) ++q;
    if (b[p] == ',') ++p;
    if (b[q] == ',') ++q;
  }
}

struct IA {
  uint64_t nc; const uint64_t* hsort; const uint32_t* jsort;   // collective events sorted by (hash, j)
  const uint32_t* perm; const uint64_t* e_gpos; const uint32_t* e_gn; const uint8_t* b;
  uint32_t* seg; uint32_t* segstart; uint32_t* first_j; JErr* err;
};

__global__ void k_j_heads(IA a) {  // seg[t] = 1 at segment heads (scanned afterwards)
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.nc) return;
  a.seg[t] = (t == 0 || a.hsort[t] != a.hsort[t - 1]) ? 1u : 0u;
}

__global__ void k_j_segs(IA a) {  // seg[t] is now the inclusive head count
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.nc) return;
  const bool head = t == 0 || a.hsort[t] != a.hsort[t - 1];
  if (head) { a.segstart[a.seg[t] - 1] = (uint32_t)t; a.first_j[a.seg[t] - 1] = a.jsort[t]; }
}

__global__ void k_j_verify(IA a) {  // exact participant-list equality with the segment head
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.nc) return;
  const uint32_t h = a.segstart[a.seg[t] - 1];
  if (h == t) return;
  const uint32_t i = a.perm[a.jsort[t]], i0 = a.perm[a.jsort[h]];
  if (a.e_gn[i] != a.e_gn[i0] || !same_group(a.b, a.e_gpos[i], a.e_gpos[i0])) atomicMax(&a.err->collide, 1ull);
}

__global__ void k_j_comm_of_seg(uint32_t ns, const uint32_t* seg_ord, uint32_t* comm_of_seg) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < ns) comm_of_seg[seg_ord[k]] = k;
}

__global__ void k_j_assign(IA a, const uint32_t* comm_of_seg, uint32_t* comm) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.nc) return;
  comm[a.jsort[t]] = comm_of_seg[a.seg[t] - 1];
}

__global__ void k_j_ccnt(uint32_t ns, const uint32_t* seg_ord, const uint32_t* first_j, const uint32_t* perm,
                         const uint32_t* e_gn, uint64_t* ccnt) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < ns) ccnt[k] = e_gn[perm[first_j[seg_ord[k]]]];
  if (k == ns) ccnt[k] = 0;
}

__global__ void k_j_members(uint32_t ns, const uint32_t* seg_ord, const uint32_t* first_j, const uint32_t* perm,
                            const uint64_t* e_gpos, const uint8_t* b, const uint64_t* coff, uint32_t* cmem) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= ns) return;
  read_group(b, e_gpos[perm[first_j[seg_ord[k]]]], cmem + coff[k], 0xFFFFFFFFu);
}

inline unsigned nb(uint64_t n, unsigned t) { return (unsigned)std::max<uint64_t>(1, (n + t - 1) / t); }

}  // namespace



// ------------------------------------------------------------------------------------- emit (J12)
namespace {

template <bool WR>
struct Out {
  uint8_t* d;
  uint64_t n;
  __device__ void ch(uint32_t x) { if (WR) d[n] = (uint8_t)x; ++n; }
  __device__ void s(const char* t) { while (*t) ch((uint8_t)*t++); }
  __device__ void u(uint64_t v) {
    char t[20];
    int k = 0;
    do { t[k++] = (char)('0' + v % 10); v /= 10; } while (v);
    while (k) ch((uint8_t)t[--k]);
  }
  __device__ void us3(int64_t ns) {  // microseconds with exactly 3 decimals
    const uint64_t a = ns < 0 ? 0ull - (uint64_t)ns : (uint64_t)ns;
    if (ns < 0) ch('-');
    u(a / 1000);
    ch('.');
    const uint32_t r = (uint32_t)(a % 1000);
    ch('0' + r / 100); ch('0' + r / 10 % 10); ch('0' + r % 10);
  }
};

struct EA {
  uint64_t N; const uint32_t* perm; const int64_t* ts; const uint32_t* dur; const uint16_t* kind; const uint16_t* meta;
  const uint32_t* comm; const uint32_t* pay; const uint32_t* rank; const uint32_t* inst; const uint64_t* coff;
  const uint32_t* cmem; uint64_t* len; const uint64_t* off; uint8_t* out;
};

template <bool WR>
__device__ uint64_t fmt_event(const EA& a, uint64_t o, uint8_t* dst) {
  Out<WR> w{dst, 0};
  const uint32_t i = a.perm[o];
  if (o) w.ch(',');
  w.ch('\n');
  const uint32_t ko = a.kind[i], m = a.meta[i], kind = ko & 7u, op = ko >> 4, iend = (ko >> 3) & 1u;
  w.s("{\"name\":\""); w.s(KNAME[kind]); w.s("\",\"cat\":\""); w.s(KNAME[kind]); w.s("\",\"ph\":\"X\",\"ts\":");
  w.us3(a.ts[i]);
  w.s(",\"dur\":"); w.us3(a.dur[i]);
  w.s(",\"pid\":"); w.u(a.rank[i]);
  w.s(",\"tid\":0,\"args\":{");
  bool first = true;
  auto sep = [&]() { if (!first) w.ch(','); first = false; };
  if (op) { sep(); w.s("\"op\":"); w.u(op); }
  if (iend) { sep(); w.s("\"iter_end\":true"); }
  if (m & 1023u) { sep(); w.s("\"mb\":"); w.u(m & 1023u); }
  if ((m >> 10) & 7u) { sep(); w.s("\"chunk\":"); w.u((m >> 10) & 7u); }
  if ((m >> 13) & 1u) { sep(); w.s("\"bwd\":1"); }
  if ((m >> 14) & 1u) { sep(); w.s("\"warmup\":1"); }
  if (kind >= 1 && kind <= 4) {
    sep();
    w.s("\"group\":[");
    const uint32_t c = a.comm[i];
    for (uint64_t q = a.coff[c]; q < a.coff[c + 1]; ++q) {
      if (q > a.coff[c]) w.ch(',');
      w.u(a.cmem[q]);
    }
    w.ch(']');
  } else if (kind >= 5) {
    sep(); w.s("\"peer\":"); w.u(a.comm[i]);
  }
  if (a.pay[i]) { sep(); w.s("\"bytes\":"); w.u(a.pay[i]); }
  if (kind) { sep(); w.s("\"related_sync_op\":"); w.u(a.inst[i]); }
  w.s("}}");
  return w.n;
}

__global__ void __launch_bounds__(128) k_e_len(EA a) {
  const uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o < a.N) a.len[o] = fmt_event<false>(a, o, nullptr);
}

__global__ void __launch_bounds__(128) k_e_write(EA a) {
  const uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o < a.N) fmt_event<true>(a, o, a.out + 16 + a.off[o]);
}

__global__ void k_e_frame(uint8_t* out, uint64_t total) {
  const char* h = "{\"traceEvents\":[";
  for (int k = 0; k < 16; ++k) out[k] = (uint8_t)h[k];
  out[total - 4] = '\n'; out[total - 3] = ']'; out[total - 2] = '}'; out[total - 1] = '\n';
}

__global__ void k_e_rank(const uint64_t* roff, uint32_t W, uint32_t* rank) {  // warp per rank
  const uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= W) return;
  for (uint64_t j = roff[r] + (threadIdx.x & 31); j < roff[r + 1]; j += 32) rank[j] = r;
}

__global__ void k_iota(uint64_t n, uint32_t* v) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) v[j] = (uint32_t)j;
}

struct XorOp {
  __device__ __forceinline__ uint8_t operator()(uint8_t a, uint8_t b) const { return a ^ b; }
};

int bits_for(uint64_t v) { int b = 1; while (b < 64 && (1ull << b) <= v) ++b; return b; }

}  // namespace

void json_release(Ctx& c) {
  JsonState* s = static_cast<JsonState*>(c.json_state);
  if (!s) return;
  DevBuf* all[] = {&s->buf, &s->docs, &s->dinfo, &s->err, &s->qm, &s->om, &s->cm, &s->par, &s->carry, &s->delta,
                   &s->esc, &s->lead, &s->ein,
                   &s->dbase, &s->wcnt, &s->wpre, &s->epos, &s->edoc, &s->e_rank, &s->e_ts, &s->e_dur, &s->e_ko,
                   &s->e_meta, &s->e_cp, &s->e_pay, &s->e_gh, &s->e_gpos, &s->e_gn, &s->keys_a, &s->keys_b,
                   &s->vals_a, &s->vals_b, &s->tmp, &s->flags, &s->sel, &s->nsel, &s->seg, &s->segstart,
                   &s->first_j, &s->seg_ord, &s->comm_of_seg, &s->ccnt, &s->coff, &s->cmem, &s->c_start, &s->c_dur,
                   &s->c_kind, &s->c_meta, &s->c_comm, &s->c_pay, &s->c_roff, &s->o_rank, &s->o_inst, &s->o_key,
                   &s->o_key2, &s->o_perm, &s->o_perm2, &s->o_len, &s->o_off, &s->out};
  for (DevBuf* b : all) b->release();
  delete s;
  c.json_state = nullptr;
}

// Parse -> event columns (device, owned by the JsonState) + host tables for scan_load_events.
scan_status json_ingest(Ctx& c, const scan_topology* topo, const uint8_t* bytes, uint64_t n, const uint64_t* doff,
                        uint32_t n_docs, uint32_t flags, scan_json_result* res, std::vector<uint64_t>& roff,
                        std::vector<uint64_t>& coff, std::vector<uint32_t>& cmem, scan_event_columns& cols) {
  *res = scan_json_result{};
  if (!topo || topo->tp < 1 || topo->pp < 1 || topo->dp < 1) { c.err = "bad topology"; return SCAN_E_INVALID_ARG; }
  const uint64_t W64 = (uint64_t)topo->tp * topo->pp * topo->dp;
  if (W64 > 65535) { c.err = "world size > 65535 unsupported"; return SCAN_E_UNSUPPORTED; }
  const uint32_t W = (uint32_t)W64;
  if (!doff || (n && !bytes)) { c.err = "missing input"; return SCAN_E_INVALID_ARG; }
  if (doff[0] != 0 || doff[n_docs] != n) { c.err = "doc_offsets must start at 0 and end at n_bytes"; return SCAN_E_INVALID_ARG; }
  for (uint32_t d = 0; d < n_docs; ++d)
    if (doff[d + 1] < doff[d]) { c.err = "doc_offsets not monotone"; return SCAN_E_INVALID_ARG; }
  JsonState& S = js(c);
  S.out_valid = false;
  const uint64_t nw = (n + 63) / 64;
  CK(S.buf.ensure(nw * 64 + 128));
  CK(cudaMemsetAsync(S.buf.p, 0, nw * 64 + 128, c.stream));
  if (n) CK(cudaMemcpyAsync(S.buf.p, bytes, n, (flags & SCAN_DEVICE_PTRS) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
  std::vector<uint64_t> hd(doff, doff + n_docs + 1);
  scan_status st;
  if ((st = upload(c, S.docs, hd))) return st;
  const JErr e0{~0ull, ~0ull, 0ull, 0ull};
  CK(S.err.ensure(sizeof(JErr)));
  CK(cudaMemcpyAsync(S.err.p, &e0, sizeof(JErr), cudaMemcpyHostToDevice, c.stream));
  CK(S.dinfo.ensure(std::max<uint32_t>(n_docs, 1) * sizeof(DocInfo)));
  const uint64_t nw1 = std::max<uint64_t>(nw, 1);
  CK(S.qm.ensure(nw1 * 8)); CK(S.om.ensure(nw1 * 8)); CK(S.cm.ensure(nw1 * 8));
  CK(S.par.ensure(nw1)); CK(S.carry.ensure(nw1)); CK(S.delta.ensure(nw1 * 4)); CK(S.dbase.ensure(nw1 * 4));
  CK(S.esc.ensure(nw1)); CK(S.lead.ensure(nw1)); CK(S.ein.ensure(nw1));
  CK(S.wcnt.ensure(nw1 * 4)); CK(S.wpre.ensure(nw1 * 4));
  const uint8_t* B = S.buf.as<uint8_t>();
  JErr* ER = S.err.as<JErr>();
  auto cub2 = [&](auto&& f) -> scan_status {
    size_t tb = 0;
    CK(f(nullptr, tb));
    CK(S.tmp.ensure(std::max<size_t>(tb, 16)));
    CK(f(S.tmp.p, tb));
    return SCAN_OK;
  };
  int launches = 0;
  JA A{B, n, S.docs.as<uint64_t>(), n_docs, nw, S.qm.as<uint64_t>(), S.om.as<uint64_t>(), S.cm.as<uint64_t>(),
       S.carry.as<uint8_t>(), S.dbase.as<int>(), S.dinfo.as<DocInfo>(), ER, S.wpre.as<uint32_t>(), S.wcnt.as<uint32_t>(),
       nullptr, nullptr};
  uint64_t n_el = 0;
  if (nw) {
    launches += timed(c, "k_j_words", [&] {
      k_j_words<<<nb(nw, 256), 256, 0, c.stream>>>(B, n, nw, S.qm.as<uint64_t>(), S.om.as<uint64_t>(), S.cm.as<uint64_t>(),
                                                   S.esc.as<uint8_t>(), S.lead.as<uint8_t>());
      return 1;
    });
    if ((st = cub2([&](void* t, size_t& tb) {  // escape state entering every word (start: not escaped)
           return cub::DeviceScan::ExclusiveScan(t, tb, S.esc.as<uint8_t>(), S.ein.as<uint8_t>(), EscOp(), (uint8_t)0,
                                                 (int64_t)nw, c.stream);
         })))
      return st;
    launches += timed(c, "k_j_escfix", [&] {
      k_j_escfix<<<nb(nw, 256), 256, 0, c.stream>>>(nw, S.qm.as<uint64_t>(), S.ein.as<uint8_t>(), S.lead.as<uint8_t>(),
                                                    S.par.as<uint8_t>());
      return 1;
    });
    if ((st = cub2([&](void* t, size_t& tb) {
           return cub::DeviceScan::ExclusiveScan(t, tb, S.par.as<uint8_t>(), S.carry.as<uint8_t>(), XorOp(), (uint8_t)0,
                                                 (int64_t)nw, c.stream);
         })))
      return st;
    launches += timed(c, "k_j_struct", [&] {
      k_j_struct<<<nb(nw, 256), 256, 0, c.stream>>>(nw, S.qm.as<uint64_t>(), S.om.as<uint64_t>(), S.cm.as<uint64_t>(),
                                                    S.carry.as<uint8_t>(), S.delta.as<int>());
      return 1;
    });
    if ((st = cub2([&](void* t, size_t& tb) {
           return cub::DeviceScan::ExclusiveSum(t, tb, S.delta.as<int>(), S.dbase.as<int>(), (int64_t)nw, c.stream);
         })))
      return st;
    launches += timed(c, "k_j_docs", [&] {
      k_j_docs1<<<nb(n_docs, 128), 128, 0, c.stream>>>(A);
      k_j_marks<<<nb(nw, 256), 256, 0, c.stream>>>(A);
      k_j_docs2<<<nb(n_docs, 128), 128, 0, c.stream>>>(A);
      k_j_arrclose<<<nb(nw, 256), 256, 0, c.stream>>>(A);
      k_j_docs3<<<nb(n_docs, 128), 128, 0, c.stream>>>(A);
      k_j_count<<<nb(nw, 256), 256, 0, c.stream>>>(A);
      return 6;
    });
    if ((st = cub2([&](void* t, size_t& tb) {
           return cub::DeviceScan::ExclusiveSum(t, tb, S.wcnt.as<uint32_t>(), S.wpre.as<uint32_t>(), (int64_t)nw, c.stream);
         })))
      return st;
    uint32_t tail[2];
    CK(cudaMemcpyAsync(&tail[0], S.wpre.as<uint32_t>() + nw - 1, 4, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(&tail[1], S.wcnt.as<uint32_t>() + nw - 1, 4, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    n_el = (uint64_t)tail[0] + tail[1];
  } else if (n_docs) {
    launches += timed(c, "k_j_docs", [&] { k_j_docs1<<<nb(n_docs, 128), 128, 0, c.stream>>>(A); return 1; });
  }
  if (n_el >= (1ull << 31)) { c.err = "more than 2^31-1 event-array elements"; return SCAN_E_UNSUPPORTED; }
  const uint64_t ne1 = std::max<uint64_t>(n_el, 1);
  CK(S.epos.ensure(ne1 * 8)); CK(S.edoc.ensure(ne1 * 4));
  CK(S.e_rank.ensure(ne1 * 4)); CK(S.e_ts.ensure(ne1 * 8)); CK(S.e_dur.ensure(ne1 * 4)); CK(S.e_ko.ensure(ne1 * 2));
  CK(S.e_meta.ensure(ne1 * 2)); CK(S.e_cp.ensure(ne1 * 4)); CK(S.e_pay.ensure(ne1 * 4)); CK(S.e_gh.ensure(ne1 * 8));
  CK(S.e_gpos.ensure(ne1 * 8)); CK(S.e_gn.ensure(ne1 * 4));
  if (n_el) {
    A.epos = S.epos.as<uint64_t>(); A.edoc = S.edoc.as<uint32_t>();
    PA P{B, S.epos.as<uint64_t>(), S.edoc.as<uint32_t>(), S.dinfo.as<DocInfo>(), n_el, W, ER,
         S.e_rank.as<uint32_t>(), S.e_ts.as<int64_t>(), S.e_dur.as<uint32_t>(), S.e_ko.as<uint16_t>(),
         S.e_meta.as<uint16_t>(), S.e_cp.as<uint32_t>(), S.e_pay.as<uint32_t>(), S.e_gh.as<uint64_t>(),
         S.e_gpos.as<uint64_t>(), S.e_gn.as<uint32_t>()};
    launches += timed(c, "k_j_place", [&] { k_j_place<<<nb(nw, 256), 256, 0, c.stream>>>(A); return 1; });
    launches += timed(c, "k_j_parse", [&] { k_j_parse<<<nb(n_el, 128), 128, 0, c.stream>>>(P); return 1; });
  }
  JErr he;
  CK(cudaMemcpyAsync(&he, S.err.p, sizeof(JErr), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  CK(cudaGetLastError());
  if (he.syn != ~0ull) {
    res->err_kind = SCAN_JSON_SYNTAX; res->err_offset = he.syn;
    c.err = "JSON syntax error at byte " + std::to_string(he.syn);
    c.launches += launches;
    return SCAN_E_SCHEMA;
  }
  if (he.sch != ~0ull) {
    res->err_kind = SCAN_JSON_SCHEMA; res->err_field = (int32_t)(he.sch & 0xFF); res->err_offset = he.sch >> 8;
    c.err = "trace schema error (field " + std::to_string(res->err_field) + ") in the element at byte " +
            std::to_string(res->err_offset);
    c.launches += launches;
    return SCAN_E_SCHEMA;
  }
  // program order: stable sort by ts, then by rank (skipped elements get rank key W: last)
  CK(S.keys_a.ensure(ne1 * 8)); CK(S.keys_b.ensure(ne1 * 8)); CK(S.vals_a.ensure(ne1 * 4)); CK(S.vals_b.ensure(ne1 * 4));
  roff.assign(W + 1, 0);
  CK(S.c_roff.ensure((W + 1) * 8));
  uint32_t* perm = S.vals_a.as<uint32_t>();
  if (n_el) {
    launches += timed(c, "k_iota", [&] { k_iota<<<nb(n_el, 256), 256, 0, c.stream>>>(n_el, S.vals_a.as<uint32_t>()); return 1; });
    if ((st = cub2([&](void* t, size_t& tb) {
           return cub::DeviceRadixSort::SortPairs(t, tb, S.e_ts.as<int64_t>(), S.keys_b.as<int64_t>(), S.vals_a.as<uint32_t>(),
                                                  S.vals_b.as<uint32_t>(), (int64_t)n_el, 0, 64, c.stream);
         })))
      return st;
    launches += timed(c, "k_j_rankkeys", [&] {
      k_j_rankkeys<<<nb(n_el, 256), 256, 0, c.stream>>>(n_el, S.vals_b.as<uint32_t>(), S.e_rank.as<uint32_t>(), W,
                                                         S.keys_a.as<uint32_t>());
      return 1;
    });
    uint32_t* rk_sorted = reinterpret_cast<uint32_t*>(S.keys_b.as<uint8_t>());
    if ((st = cub2([&](void* t, size_t& tb) {
           return cub::DeviceRadixSort::SortPairs(t, tb, S.keys_a.as<uint32_t>(), rk_sorted, S.vals_b.as<uint32_t>(), perm,
                                                  (int64_t)n_el, 0, bits_for(W), c.stream);
         })))
      return st;
    launches += timed(c, "k_j_roff", [&] { k_j_roff<<<nb(W + 1, 128), 128, 0, c.stream>>>(n_el, rk_sorted, W, S.c_roff.as<uint64_t>()); return 1; });
    CK(cudaMemcpyAsync(roff.data(), S.c_roff.p, (W + 1) * 8, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
  }
  const uint64_t N = roff[W];
  res->n_events = N;
  res->n_skipped = n_el - N;
  const uint64_t N1 = std::max<uint64_t>(N, 1);
  CK(S.c_start.ensure(N1 * 8)); CK(S.c_dur.ensure(N1 * 4)); CK(S.c_kind.ensure(N1 * 2)); CK(S.c_meta.ensure(N1 * 2));
  CK(S.c_comm.ensure(N1 * 4)); CK(S.c_pay.ensure(N1 * 4)); CK(S.flags.ensure(N1)); CK(S.keys_a.ensure(N1 * 8));
  uint64_t nC = 0;
  coff.assign(1, 0);
  cmem.clear();
  if (N) {
    GA G{N, perm, S.e_ts.as<int64_t>(), S.e_dur.as<uint32_t>(), S.e_ko.as<uint16_t>(), S.e_meta.as<uint16_t>(),
         S.e_cp.as<uint32_t>(), S.e_pay.as<uint32_t>(), S.e_gh.as<uint64_t>(), S.c_start.as<int64_t>(),
         S.c_dur.as<uint32_t>(), S.c_kind.as<uint16_t>(), S.c_meta.as<uint16_t>(), S.c_comm.as<uint32_t>(),
         S.c_pay.as<uint32_t>(), S.flags.as<uint8_t>(), S.keys_a.as<uint64_t>()};
    launches += timed(c, "k_j_gather", [&] { k_j_gather<<<nb(N, 256), 256, 0, c.stream>>>(G); return 1; });
    // collectives in program order: (hash, j), sorted by hash (stable: ascending j within a hash)
    CK(S.sel.ensure(N1 * 4)); CK(S.nsel.ensure(16)); CK(S.vals_b.ensure(N1 * 4)); CK(S.keys_b.ensure(N1 * 8));
    CK(S.seg.ensure(N1 * 8)); CK(S.first_j.ensure(N1 * 4));
    uint64_t* hsel = reinterpret_cast<uint64_t*>(S.seg.as<uint8_t>());  // temporary: selected hashes
    if ((st = cub2([&](void* t, size_t& tb) {
           return cub::DeviceSelect::Flagged(t, tb, cub::CountingInputIterator<uint32_t>(0), S.flags.as<uint8_t>(),
                                             S.sel.as<uint32_t>(), S.nsel.as<uint64_t>(), (int64_t)N, c.stream);
         })))
      return st;
    if ((st = cub2([&](void* t, size_t& tb) {
           return cub::DeviceSelect::Flagged(t, tb, S.keys_a.as<uint64_t>(), S.flags.as<uint8_t>(), hsel,
                                             S.nsel.as<uint64_t>(), (int64_t)N, c.stream);
         })))
      return st;
    CK(cudaMemcpyAsync(&nC, S.nsel.p, 8, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    if (nC) {
      uint64_t* hsort = S.keys_b.as<uint64_t>();
      uint32_t* jsort = S.vals_b.as<uint32_t>();
      if ((st = cub2([&](void* t, size_t& tb) {
             return cub::DeviceRadixSort::SortPairs(t, tb, hsel, hsort, S.sel.as<uint32_t>(), jsort, (int64_t)nC, 0, 64, c.stream);
           })))
        return st;
      CK(S.segstart.ensure(nC * 4)); CK(S.seg_ord.ensure(nC * 4)); CK(S.comm_of_seg.ensure(nC * 4));
      uint32_t* seg = S.sel.as<uint32_t>();  // reuse: the selected j are in jsort now
      IA I{nC, hsort, jsort, perm, S.e_gpos.as<uint64_t>(), S.e_gn.as<uint32_t>(), B, seg, S.segstart.as<uint32_t>(),
           S.first_j.as<uint32_t>(), ER};
      launches += timed(c, "k_j_heads", [&] { k_j_heads<<<nb(nC, 256), 256, 0, c.stream>>>(I); return 1; });
      if ((st = cub2([&](void* t, size_t& tb) {
             return cub::DeviceScan::InclusiveSum(t, tb, seg, seg, (int64_t)nC, c.stream);
           })))
        return st;
      uint32_t ns = 0;
      CK(cudaMemcpyAsync(&ns, seg + nC - 1, 4, cudaMemcpyDeviceToHost, c.stream));
      launches += timed(c, "k_j_segs", [&] {
        k_j_segs<<<nb(nC, 256), 256, 0, c.stream>>>(I);
        k_j_verify<<<nb(nC, 256), 256, 0, c.stream>>>(I);
        return 2;
      });
      CK(cudaStreamSynchronize(c.stream));
      // segments in order of first use -> communicator ids
      uint32_t* fsorted = S.segstart.as<uint32_t>();  // segstart no longer needed after k_j_verify
      CK(S.keys_a.ensure(std::max<uint64_t>(ns, 1) * 4));
      uint32_t* sid = S.keys_a.as<uint32_t>();
      launches += timed(c, "k_iota", [&] { k_iota<<<nb(ns, 256), 256, 0, c.stream>>>(ns, sid); return 1; });
      if ((st = cub2([&](void* t, size_t& tb) {
             return cub::DeviceRadixSort::SortPairs(t, tb, S.first_j.as<uint32_t>(), fsorted, sid, S.seg_ord.as<uint32_t>(),
                                                    (int64_t)ns, 0, 32, c.stream);
           })))
        return st;
      CK(S.ccnt.ensure((ns + 1) * 8)); CK(S.coff.ensure((ns + 1) * 8));
      launches += timed(c, "k_j_intern", [&] {
        k_j_comm_of_seg<<<nb(ns, 256), 256, 0, c.stream>>>(ns, S.seg_ord.as<uint32_t>(), S.comm_of_seg.as<uint32_t>());
        k_j_assign<<<nb(nC, 256), 256, 0, c.stream>>>(I, S.comm_of_seg.as<uint32_t>(), S.c_comm.as<uint32_t>());
        // first_j of segment s (sorted) = fsorted[k] for the k-th communicator
        k_j_ccnt<<<nb(ns + 1, 256), 256, 0, c.stream>>>(ns, S.seg_ord.as<uint32_t>(), S.first_j.as<uint32_t>(), perm,
                                                         S.e_gn.as<uint32_t>(), S.ccnt.as<uint64_t>());
        return 3;
      });
      if ((st = cub2([&](void* t, size_t& tb) {
             return cub::DeviceScan::ExclusiveSum(t, tb, S.ccnt.as<uint64_t>(), S.coff.as<uint64_t>(), (int64_t)ns + 1, c.stream);
           })))
        return st;
      coff.resize(ns + 1);
      CK(cudaMemcpyAsync(coff.data(), S.coff.p, (ns + 1) * 8, cudaMemcpyDeviceToHost, c.stream));
      CK(cudaStreamSynchronize(c.stream));
      CK(S.cmem.ensure(std::max<uint64_t>(coff[ns], 1) * 4));
      launches += timed(c, "k_j_members", [&] {
        k_j_members<<<nb(ns, 128), 128, 0, c.stream>>>(ns, S.seg_ord.as<uint32_t>(), S.first_j.as<uint32_t>(), perm,
                                                       S.e_gpos.as<uint64_t>(), B, S.coff.as<uint64_t>(), S.cmem.as<uint32_t>());
        return 1;
      });
      cmem.resize(coff[ns]);
      if (!cmem.empty()) CK(cudaMemcpyAsync(cmem.data(), S.cmem.p, cmem.size() * 4, cudaMemcpyDeviceToHost, c.stream));
      CK(cudaMemcpyAsync(&he, S.err.p, sizeof(JErr), cudaMemcpyDeviceToHost, c.stream));
      CK(cudaStreamSynchronize(c.stream));
      CK(cudaGetLastError());
      if (he.collide) { c.err = "64-bit participant-list hash collision"; c.launches += launches; return SCAN_E_UNSUPPORTED; }
      res->n_comms = ns;
    }
  }
  c.launches += launches;
  cols = scan_event_columns{N, roff.data(), S.c_start.as<int64_t>(), S.c_dur.as<uint32_t>(), S.c_kind.as<uint16_t>(),
                            S.c_meta.as<uint16_t>(), S.c_comm.as<uint32_t>(), S.c_pay.as<uint32_t>()};
  return SCAN_OK;
}

scan_status json_emit(Ctx& c, uint32_t flags, bool reuse) {
  JsonState& S = js(c);
  if (reuse && S.out_valid && S.out_flags == flags && S.out_gen == c.gen) return SCAN_OK;
  S.out_valid = false;
  const uint64_t N = c.N;
  const uint32_t W = (uint32_t)c.W;
  const int64_t* ts = (flags & SCAN_EMIT_ALIGNED) ? c.al_start.as<int64_t>() : c.d_start;
  scan_status st = ensure_tiles(c);
  if (st) return st;
  const uint64_t N1 = std::max<uint64_t>(N, 1);
  CK(S.o_inst.ensure(N1 * 4)); CK(S.o_rank.ensure(N1 * 4)); CK(S.o_key2.ensure(N1 * 8)); CK(S.o_perm.ensure(N1 * 4));
  CK(S.o_perm2.ensure(N1 * 4)); CK(S.o_len.ensure(N1 * 8)); CK(S.o_off.ensure(N1 * 8));
  auto cub2 = [&](auto&& f) -> scan_status {
    size_t tb = 0;
    CK(f(nullptr, tb));
    CK(S.tmp.ensure(std::max<size_t>(tb, 16)));
    CK(f(S.tmp.p, tb));
    return SCAN_OK;
  };
  uint64_t total = 16 + 4;
  if (N) {
    launch_expand_events(c, SCAN_OUT_EV_INST, S.o_inst.p);
    flush_fills(c);
    k_e_rank<<<nb((uint64_t)W * 32, 256), 256, 0, c.stream>>>(c.rank_off.as<uint64_t>(), W, S.o_rank.as<uint32_t>());
    k_iota<<<nb(N, 256), 256, 0, c.stream>>>(N, S.o_perm2.as<uint32_t>());
    if ((st = cub2([&](void* t, size_t& tb) {
           return cub::DeviceRadixSort::SortPairs(t, tb, ts, S.o_key2.as<int64_t>(), S.o_perm2.as<uint32_t>(),
                                                  S.o_perm.as<uint32_t>(), (int64_t)N, 0, 64, c.stream);
         })))
      return st;
    EA a{N, S.o_perm.as<uint32_t>(), ts, c.d_dur, c.d_kind, c.d_meta, c.d_comm, c.d_pay, S.o_rank.as<uint32_t>(),
         S.o_inst.as<uint32_t>(), c.coff.as<uint64_t>(), c.cmem.as<uint32_t>(), S.o_len.as<uint64_t>(),
         S.o_off.as<uint64_t>(), nullptr};
    k_e_len<<<nb(N, 128), 128, 0, c.stream>>>(a);
    if ((st = cub2([&](void* t, size_t& tb) {
           return cub::DeviceScan::ExclusiveSum(t, tb, S.o_len.as<uint64_t>(), S.o_off.as<uint64_t>(), (int64_t)N, c.stream);
         })))
      return st;
    uint64_t lo[2];
    CK(cudaMemcpyAsync(&lo[0], S.o_off.as<uint64_t>() + N - 1, 8, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(&lo[1], S.o_len.as<uint64_t>() + N - 1, 8, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    total += lo[0] + lo[1];
    CK(S.out.ensure(total));
    a.out = S.out.as<uint8_t>();
    k_e_write<<<nb(N, 128), 128, 0, c.stream>>>(a);
    c.launches += 6;
  } else {
    CK(S.out.ensure(total));
  }
  k_e_frame<<<1, 1, 0, c.stream>>>(S.out.as<uint8_t>(), total);
  CK(cudaStreamSynchronize(c.stream));
  CK(cudaGetLastError());
  S.out_bytes = total; S.out_flags = flags; S.out_gen = c.gen; S.out_valid = true;
  return SCAN_OK;
}

}  // namespace ms

using namespace ms;

extern "C" {

scan_status scan_ingest_json(scan_ctx* ctx, const scan_topology* topo, const uint8_t* bytes, uint64_t n_bytes,
                             const uint64_t* doc_offsets, uint32_t n_docs, uint32_t flags, scan_json_result* out) {
  if (!ctx) return SCAN_E_INVALID_ARG;
  Ctx& c = ctx->c;
  CK(cudaSetDevice(c.device));
  if (c.n_shards > 1) { c.err = "JSON ingest on a sharded context is unsupported"; return SCAN_E_UNSUPPORTED; }
  scan_json_result r{};
  std::vector<uint64_t> roff, coff;
  std::vector<uint32_t> cmem;
  scan_event_columns cols{};
  c.loaded = c.matched = c.detected = c.localized = false;
  scan_status st = json_ingest(c, topo, bytes, n_bytes, doc_offsets, n_docs, flags, &r, roff, coff, cmem, cols);
  if (out) *out = r;
  if (st) return st;
  const scan_comm_table ct{(uint32_t)(coff.size() - 1), coff.data(), cmem.empty() ? nullptr : cmem.data()};
  st = scan_load_events(ctx, topo, &ct, &cols, SCAN_DEVICE_PTRS | (flags & SCAN_STRICT));
  return st;
}

scan_status scan_loaded_column(scan_ctx* ctx, int column, void* dst, uint64_t dst_bytes, int dst_is_device, uint64_t* bytes) {
  if (!ctx || !bytes) return SCAN_E_INVALID_ARG;
  Ctx& c = ctx->c;
  if (!c.loaded) { c.err = "nothing loaded"; return SCAN_E_ORDER; }
  CK(cudaSetDevice(c.device));
  const void* src = nullptr;
  uint64_t nbytes = 0;
  bool host = false;
  switch (column) {
    case 0: src = c.d_start; nbytes = c.d_start ? c.N * 8 : 0; break;
    case 1: src = c.d_dur; nbytes = c.N * 4; break;
    case 2: src = c.d_kind; nbytes = c.N * 2; break;
    case 3: src = c.d_meta; nbytes = c.N * 2; break;
    case 4: src = c.d_comm; nbytes = c.N * 4; break;
    case 5: src = c.d_pay; nbytes = c.N * 4; break;
    case 6: src = c.h_rank_off.data(); nbytes = c.h_rank_off.size() * 8; host = true; break;
    case 7: src = c.h_coff.data(); nbytes = c.h_coff.size() * 8; host = true; break;
    case 8: src = c.h_cmem.data(); nbytes = c.h_cmem.size() * 4; host = true; break;
    default: c.err = "bad column"; return SCAN_E_INVALID_ARG;
  }
  if (column == 0 && !c.d_start) { c.err = "no start_ns loaded"; return SCAN_E_INVALID_ARG; }
  *bytes = nbytes;
  if (!dst) return SCAN_OK;
  if (dst_bytes < nbytes) { c.err = "destination too small"; return SCAN_E_INVALID_ARG; }
  if (!nbytes) return SCAN_OK;
  const cudaMemcpyKind k = host ? (dst_is_device ? cudaMemcpyHostToDevice : cudaMemcpyHostToHost)
                                : (dst_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost);
  CK(cudaMemcpyAsync(dst, src, nbytes, k, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  return SCAN_OK;
}

scan_status scan_emit_chrome(scan_ctx* ctx, uint32_t flags, void* dst, uint64_t dst_bytes, int dst_is_device, uint64_t* n_bytes) {
  if (!ctx || !n_bytes) return SCAN_E_INVALID_ARG;
  Ctx& c = ctx->c;
  CK(cudaSetDevice(c.device));
  // a sharded context emits its own iteration block (job-wide instance ids); the job's document is the
  // shards' documents merged by (ts, pid, shard order)
  if (c.stream_mode) { c.err = "emit is unavailable on stream contexts"; return SCAN_E_UNSUPPORTED; }
  if (!c.loaded || !c.matched) { c.err = "emit needs a loaded and matched trace"; return SCAN_E_ORDER; }
  if (flags & ~SCAN_EMIT_ALIGNED) { c.err = "unknown emit flags"; return SCAN_E_INVALID_ARG; }
  if ((flags & SCAN_EMIT_ALIGNED) && !c.aligned) { c.err = "SCAN_EMIT_ALIGNED needs scan_align"; return SCAN_E_ORDER; }
  if (!(flags & SCAN_EMIT_ALIGNED) && !c.d_start) { c.err = "emit needs start_ns at load"; return SCAN_E_INVALID_ARG; }
  scan_status st = json_emit(c, flags, dst != nullptr);  // a size query (dst NULL) always builds
  if (st) return st;
  JsonState& S = js(c);
  *n_bytes = S.out_bytes;
  if (!dst) return SCAN_OK;
  if (dst_bytes < S.out_bytes) { c.err = "destination too small"; return SCAN_E_INVALID_ARG; }
  CK(cudaMemcpyAsync(dst, S.out.p, S.out_bytes, dst_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  return SCAN_OK;
}

}  // extern "C"
