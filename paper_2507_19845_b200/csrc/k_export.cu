// k_export.cu — untimed expansion of the compact native layouts to the event-order / instance
// arrays of the export API (used by tests and users that want per-event arrays).
#include "internal.cuh"

namespace ms {

struct ExpArgs {
  const uint32_t* tile_rank; const uint64_t* tile_start; const uint64_t* rank_off;
  const uint16_t* kind; uint64_t N; uint64_t n_tiles; int TP, DP;
  const uint32_t* t_commpre; const uint64_t* r_comm_off; const uint64_t* r_comp_off; const uint64_t* r_bits_off;
  const uint32_t* inst_c; const uint32_t* wait_c; const uint32_t* bits; const uint32_t* cref; const uint32_t* cl_J;
  int which; void* dst;
};

__global__ void __launch_bounds__(256) k_expand(ExpArgs a) {
  const uint64_t tile = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (tile >= a.n_tiles) return;
  const uint32_t lane = lane_id();
  const uint32_t r = a.tile_rank[tile];
  const uint64_t rstart = a.rank_off[r];
  const uint64_t s = a.tile_start[tile];
  const uint64_t e = min(s + (uint64_t)TILE_EV, a.rank_off[r + 1]);
  uint32_t comm_carry = a.t_commpre[tile];
  const uint64_t co = a.r_comm_off[r], po = a.r_comp_off[r];
  uint32_t J = 0;
  if (a.DP >= 2 && a.cl_J) J = a.cl_J[(r / (uint32_t)(a.TP * a.DP)) * a.TP + r % a.TP];
  for (uint64_t base = s & ~7ull; base < e; base += 256) {
    const uint64_t g = base + 8ull * lane;
    uint16_t ko[8];
    load8_u16(a.kind, g, a.N, ko);
    uint32_t valid = 0, commm = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint64_t ev = g + q;
      if (ev < s || ev >= e) continue;
      valid |= 1u << q;
      if (ko[q] & 7u) commm |= 1u << q;
    }
    uint32_t ctot;
    const uint32_t cex = warp_excl_scan(__popc(commm), ctot) + comm_carry;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (!((valid >> q) & 1u)) continue;
      const uint64_t ev = g + q;
      const uint32_t cb = cex + __popc(commm & ((1u << q) - 1u));
      const bool isc = (commm >> q) & 1u;
      const uint32_t j = (uint32_t)(ev - rstart) - cb;
      switch (a.which) {
        case SCAN_OUT_EV_INST: ((uint32_t*)a.dst)[ev] = isc ? a.inst_c[co + cb] : NONE32; break;
        case SCAN_OUT_EV_WAIT: ((uint32_t*)a.dst)[ev] = (isc && a.wait_c) ? a.wait_c[co + cb] : 0u; break;
        case SCAN_OUT_EV_SLOW: {
          uint8_t v = 0;
          if (!isc && j < J && a.bits) v = (a.bits[a.r_bits_off[r] + (j >> 5)] >> (j & 31)) & 1u;
          ((uint8_t*)a.dst)[ev] = v;
          break;
        }
        case SCAN_OUT_EV_REF: ((uint32_t*)a.dst)[ev] = (!isc && j < J && a.cref) ? a.cref[po + j] : NONE32; break;
        default: break;
      }
    }
    comm_carry += ctot;
  }
}

int launch_expand_events(Ctx& c, scan_output which, void* dst) {
  if (c.n_tiles == 0) return 0;
  ExpArgs a{c.tile_rank.as<uint32_t>(), c.tile_start.as<uint64_t>(), c.rank_off.as<uint64_t>(), c.d_kind, c.N,
            c.n_tiles, c.TP, c.DP, c.t_commpre.as<uint32_t>(), c.r_comm_off.as<uint64_t>(), c.r_comp_off.as<uint64_t>(),
            c.r_bits_off.as<uint64_t>(), c.inst_c.as<uint32_t>(), c.localized ? c.wait_c.as<uint32_t>() : nullptr,
            c.detected ? c.bits.as<uint32_t>() : nullptr, (c.detected && c.dcfg.want_ref) ? c.cref.as<uint32_t>() : nullptr,
            c.detected ? c.cl_J.as<uint32_t>() : nullptr, (int)which, dst};
  k_expand<<<(unsigned)((c.n_tiles + 7) / 8), 256, 0, c.stream>>>(a);
  return 1;
}

__global__ void k_inst_export(uint64_t n_inst, uint64_t NCH, uint32_t n_comms, const uint64_t* ch_base,
                              const uint64_t* ch_slot, const uint32_t* ch_nmin, const uint64_t* coff, const uint32_t* cmem,
                              const uint32_t* nsend, const uint32_t* nrecv, const uint32_t* r_nkeys, const uint32_t* r_keys,
                              const uint32_t* r_cnt, const uint4* rec, const uint4* slots,
                              const uint64_t* kshift, int which, void* dst) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_inst; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t ch = upper_bound_u64(ch_base, NCH + 1, i) - 1;
    const uint64_t k = i - ch_base[ch];
    const uint64_t kl = kshift ? k - kshift[ch] : k;  // occurrence index among this shard's events
    const uint4 rc = rec[i];
    const bool isp = ch >= n_comms;
    switch (which) {
      case SCAN_OUT_IN_CHANNEL: ((uint32_t*)dst)[i] = (uint32_t)ch; break;
      case SCAN_OUT_IN_K: ((uint32_t*)dst)[i] = (uint32_t)k; break;
      case SCAN_OUT_IN_FLAGS: ((uint8_t*)dst)[i] = (uint8_t)(rc.w & 0xFFu); break;
      case SCAN_OUT_IN_DMIN: ((uint32_t*)dst)[i] = rc.x; break;
      case SCAN_OUT_IN_DMAX: ((uint32_t*)dst)[i] = rc.y; break;
      case SCAN_OUT_IN_LAST: ((uint32_t*)dst)[i] = rc.z; break;
      case SCAN_OUT_IN_NPRESENT: {
        uint32_t n = 0;
        if (!isp) {
          const uint32_t nm = (uint32_t)(coff[ch + 1] - coff[ch]);
          if (kl < ch_nmin[ch]) n = nm;
          else
            for (uint32_t q = 0; q < nm; ++q) {
              const uint32_t m = cmem[coff[ch] + q];
              const uint32_t C = r_nkeys[m];
              const uint32_t p = lower_bound_u32(r_keys + (uint64_t)m * RCAP, C, (uint32_t)ch);
              if (p < C && r_keys[(uint64_t)m * RCAP + p] == (uint32_t)ch && r_cnt[(uint64_t)m * RCAP + p] > kl) ++n;
            }
        } else {
          n = (nsend[ch - n_comms] > kl) + (nrecv[ch - n_comms] > kl);
        }
        ((uint32_t*)dst)[i] = n;
        break;
      }
      case SCAN_OUT_IN_PAYLOAD: {
        uint32_t v = 0;
        if (isp) {
          const uint64_t sb = ch_slot[ch] + k * 2;
          if (nsend[ch - n_comms] > kl) v = slots[sb].w;
          else if (nrecv[ch - n_comms] > kl) v = slots[sb + 1].w;
        }
        ((uint32_t*)dst)[i] = v;
        break;
      }
      default: break;
    }
  }
}

int launch_instance_export(Ctx& c, scan_output which, void* dst) {
  if (c.n_inst == 0) return 0;
  unsigned blocks = (unsigned)std::min<uint64_t>((c.n_inst + 255) / 256, 148ull * 16);
  // sharded: global channel tables; member counts are this shard's (valid for its own instance ranges)
  const bool sh = c.n_shards > 1;
  k_inst_export<<<blocks, 256, 0, c.stream>>>(c.n_inst, c.NCH, c.n_comms, (sh ? c.g_base : c.ch_base).as<uint64_t>(),
                                              (sh ? c.g_slot : c.ch_slot).as<uint64_t>(),
                                              c.ch_nmin.as<uint32_t>(), c.coff.as<uint64_t>(), c.cmem.as<uint32_t>(),
                                              c.ch_nsend.as<uint32_t>(), c.ch_nrecv.as<uint32_t>(), c.r_nkeys.as<uint32_t>(),
                                              c.r_keys.as<uint32_t>(), c.r_cnt.as<uint32_t>(), c.inst_rec.as<uint4>(),
                                              c.slots.as<uint4>(), sh ? c.g_k0.as<uint64_t>() : nullptr,
                                              (int)which, dst);
  return 1;
}

}  // namespace ms
