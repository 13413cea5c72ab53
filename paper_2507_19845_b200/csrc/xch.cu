// xch.cu — the exchange layer of the sharded analysis (row A9, shard.cu): the four collective shapes
// scan_analyze uses between shards (all-gather, grouped send / recv, grouped all-reduce sum) on one of
// two back-ends:
//   * NCCL over NVLink / NVSwitch: one process per GPU, the context's own communicator (production);
//   * an in-process group: G shard contexts driven by G host threads of one process, on one or more
//     GPUs of that process. Collectives rendezvous on a host barrier and move data with device copies
//     and a summing kernel. It exists so the sharded path (its numbering, exchanges and fix-ups) runs
//     and is checked against the oracle on a single-GPU box (tests/test_gpu_multi_local.py); it is not
//     a performance path.
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.cuh"

namespace ms {

struct LocalGroup {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> ptr;          // all-gather: each rank's send buffer
  std::vector<std::vector<XOp>> ops;     // grouped ops published by each rank
  void barrier() {
    std::unique_lock<std::mutex> l(m);
    const uint64_t g = gen;
    if (++arrived == n) { arrived = 0; ++gen; cv.notify_all(); }
    else cv.wait(l, [&] { return gen != g; });
  }
};

namespace {

constexpr int XMAX = 16;  // shards of an in-process group
struct Ptrs { const void* p[XMAX]; };

template <class T>
__global__ void k_xsum(T* out, Ptrs in, int n_in, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    T s = 0;
    for (int r = 0; r < n_in; ++r) s += static_cast<const T*>(in.p[r])[i];
    out[i] = s;
  }
}

size_t xsize(int type) { return type == XU8 ? 1 : (type == XU32 ? 4 : 8); }

ncclDataType_t ntype(int type) {
  return type == XU8 ? ncclUint8 : (type == XU32 ? ncclUint32 : (type == XU64 ? ncclUint64 : ncclFloat64));
}

int lerr(cudaError_t e) { return e == cudaSuccess ? 0 : 1000 + (int)e; }

}  // namespace

const char* xch_error(int rc) {
  if (rc >= 1000) return cudaGetErrorString((cudaError_t)(rc - 1000));
  return ncclGetErrorString((ncclResult_t)rc);
}

int xch_allgather(Ctx& c, const void* send, void* recv, size_t n_u32) {
  if (c.nccl) return (int)ncclAllGather(send, recv, n_u32, ncclUint32, (ncclComm_t)c.nccl, c.stream);
  LocalGroup& g = *static_cast<LocalGroup*>(c.lgroup);
  cudaError_t e = cudaStreamSynchronize(c.stream);  // the send buffer is final
  g.ptr[c.shard] = send;
  g.barrier();
  for (int r = 0; r < g.n && e == cudaSuccess; ++r)
    e = cudaMemcpyAsync(static_cast<uint8_t*>(recv) + (size_t)r * n_u32 * 4, g.ptr[r], n_u32 * 4, cudaMemcpyDefault, c.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
  g.barrier();  // every rank has read every send buffer before any of them changes
  return lerr(e);
}

void xch_group_start(Ctx& c) {
  if (c.nccl) { ncclGroupStart(); return; }
  c.xops.clear();
}

void xch_send(Ctx& c, const void* p, size_t n_u32, int peer) {
  if (c.nccl) { ncclSend(p, n_u32, ncclUint32, peer, (ncclComm_t)c.nccl, c.stream); return; }
  c.xops.push_back({0, p, nullptr, n_u32 * 4, XU32, peer});
}

void xch_recv(Ctx& c, void* p, size_t n_u32, int peer) {
  if (c.nccl) { ncclRecv(p, n_u32, ncclUint32, peer, (ncclComm_t)c.nccl, c.stream); return; }
  c.xops.push_back({1, nullptr, p, n_u32 * 4, XU32, peer});
}

void xch_allreduce(Ctx& c, void* p, size_t n, int type) {
  if (c.nccl) { ncclAllReduce(p, p, n, ntype(type), ncclSum, (ncclComm_t)c.nccl, c.stream); return; }
  c.xops.push_back({2, p, p, n, type, -1});
}

int xch_group_end(Ctx& c) {
  if (c.nccl) return (int)ncclGroupEnd();
  LocalGroup& g = *static_cast<LocalGroup*>(c.lgroup);
  const int me = c.shard;
  cudaError_t e = cudaStreamSynchronize(c.stream);
  g.ops[me] = c.xops;
  g.barrier();
  // point-to-point: the k-th receive from s takes the k-th send of s addressed to this rank
  std::vector<int> taken(g.n, 0);
  for (const XOp& o : c.xops) {
    if (o.kind != 1 || e != cudaSuccess) continue;
    int k = taken[o.peer]++;
    const XOp* src = nullptr;
    for (const XOp& so : g.ops[o.peer])
      if (so.kind == 0 && so.peer == me && k-- == 0) { src = &so; break; }
    if (!src || src->n != o.n) { e = cudaErrorInvalidValue; break; }
    e = cudaMemcpyAsync(o.recv, src->send, o.n, cudaMemcpyDefault, c.stream);
  }
  // all-reduce (sum): op i of every rank has the same shape; sums into a private buffer first, the
  // in-place overwrite only after every rank has read every input
  std::vector<size_t> toff;
  size_t tot = 0;
  for (const XOp& o : c.xops)
    if (o.kind == 2) { toff.push_back(tot); tot += (o.n * xsize(o.type) + 255) & ~size_t(255); }
  if (tot && e == cudaSuccess) e = c.xtmp.ensure(tot);
  size_t ai = 0;
  for (size_t i = 0; i < c.xops.size() && e == cudaSuccess; ++i) {
    const XOp& o = c.xops[i];
    if (o.kind != 2) continue;
    Ptrs in{};
    int idx = 0;
    for (int r = 0; r < g.n; ++r) {
      int seen = 0;
      for (const XOp& ro : g.ops[r])
        if (ro.kind == 2 && seen++ == (int)ai) { in.p[idx++] = ro.send; break; }
    }
    void* out = static_cast<uint8_t*>(c.xtmp.p) + toff[ai];
    const unsigned blocks = (unsigned)std::min<uint64_t>((o.n + 255) / 256, 1024);
    if (o.n) {
      if (o.type == XU8) k_xsum<uint8_t><<<blocks, 256, 0, c.stream>>>(static_cast<uint8_t*>(out), in, idx, o.n);
      else if (o.type == XU32) k_xsum<uint32_t><<<blocks, 256, 0, c.stream>>>(static_cast<uint32_t*>(out), in, idx, o.n);
      else if (o.type == XU64) k_xsum<unsigned long long><<<blocks, 256, 0, c.stream>>>(static_cast<unsigned long long*>(out), in, idx, o.n);
      else k_xsum<double><<<blocks, 256, 0, c.stream>>>(static_cast<double*>(out), in, idx, o.n);
      e = cudaGetLastError();
    }
    ++ai;
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
  g.barrier();  // all reads of the send buffers are done
  ai = 0;
  for (const XOp& o : c.xops) {
    if (o.kind != 2) continue;
    if (e == cudaSuccess && o.n)
      e = cudaMemcpyAsync(o.recv, static_cast<uint8_t*>(c.xtmp.p) + toff[ai], o.n * xsize(o.type), cudaMemcpyDefault, c.stream);
    ++ai;
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
  g.barrier();
  c.xops.clear();
  return lerr(e);
}

}  // namespace ms

using namespace ms;

struct scan_local_group { ms::LocalGroup g; };

extern "C" {

scan_status scan_local_group_create(scan_local_group** out, int n_shards) {
  if (!out || n_shards < 1 || n_shards > 16) return SCAN_E_INVALID_ARG;
  auto* lg = new scan_local_group();
  lg->g.n = n_shards;
  lg->g.ptr.assign(n_shards, nullptr);
  lg->g.ops.assign(n_shards, {});
  *out = lg;
  return SCAN_OK;
}

void scan_local_group_destroy(scan_local_group* group) { delete group; }

scan_status scan_create_sharded_local(scan_ctx** out, int cuda_device, void* cuda_stream, scan_local_group* group, int shard) {
  if (!out || !group || shard < 0 || shard >= group->g.n) return SCAN_E_INVALID_ARG;
  scan_status st = scan_create(out, cuda_device, cuda_stream);
  if (st) return st;
  Ctx& c = (*out)->c;
  c.n_shards = group->g.n; c.shard = shard;
  c.lgroup = &group->g;
  return SCAN_OK;
}

}  // extern "C"
