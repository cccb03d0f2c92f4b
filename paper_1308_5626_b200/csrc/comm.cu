// comm.cu -- the communicator behind psp_comm: NCCL over NVLink/NVSwitch for real ranks (one
// process per GPU), and an in-process loopback group for testing the multi-rank code path with
// several contexts on ONE device (host-mediated: every collective synchronises the caller's
// stream, meets the other ranks at a host barrier and copies device buffers with cudaMemcpy;
// no kernel ever waits on another rank's kernel).
//
// Collectives used by the hot path:
//   allreduce      -- Arnoldi dots / norms (sum), MREP gate statistics (max/min/sum)
//   sendrecv       -- slab halos: one plane for the stencil, d rows x m probes for MREP,
//                     the fixed-point state of the banded factorisation
//   allgather      -- per-rank affine maps / states of the partitioned banded sweeps
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <condition_variable>
#include <memory>
#include <mutex>
#include <vector>

#include "internal.h"

namespace {

// NCCL is bound at first use (dlopen of libnccl.so.2), not at load time: a process that uses
// the library on one GPU never loads NCCL, and in a torch.distributed job the already-loaded
// libnccl.so.2 of torch is the one bound (loading the system copy first would shadow torch's).
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
};
const NcclApi& nccl() {
  static NcclApi a;
  static bool tried = false;
  if (tried) return a;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // torch's copy, if loaded
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW);
  if (!h) return a;
  auto sym = [&](const char* n) { return dlsym(h, n); };
  a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
  a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
  a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
  a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
  a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
  a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
  a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
  a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
  a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
  a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.AllGather && a.Send && a.Recv &&
         a.GroupStart && a.GroupEnd;
  return a;
}

ncclRedOp_t nccl_op(int op) { return op == 1 ? ncclMax : (op == 2 ? ncclMin : ncclSum); }

struct NcclComm : psp_comm {
  ncclComm_t c = nullptr;
  ~NcclComm() override {
    if (c && nccl().ok) nccl().CommDestroy(c);
  }
  int allreduce(double* d, size_t count, int op, cudaStream_t s) override {
    if (!c) return nranks == 1 ? 0 : 1;            // one rank without NCCL: the identity
    return nccl().AllReduce(d, d, count, ncclDouble, nccl_op(op), c, s) == ncclSuccess ? 0 : 1;
  }
  int sendrecv(const double* send_lo, double* recv_lo, size_t n_lo, const double* send_hi,
               double* recv_hi, size_t n_hi, cudaStream_t s) override {
    const NcclApi& A = nccl();
    if (A.GroupStart() != ncclSuccess) return 1;
    if (rank > 0 && n_lo) {
      A.Send(send_lo, n_lo, ncclDouble, rank - 1, c, s);
      A.Recv(recv_lo, n_lo, ncclDouble, rank - 1, c, s);
    }
    if (rank < nranks - 1 && n_hi) {
      A.Send(send_hi, n_hi, ncclDouble, rank + 1, c, s);
      A.Recv(recv_hi, n_hi, ncclDouble, rank + 1, c, s);
    }
    return A.GroupEnd() == ncclSuccess ? 0 : 1;
  }
  int allgather(const double* send, double* recv, size_t count, cudaStream_t s) override {
    if (!c) return (nranks == 1 && cudaMemcpyAsync(recv, send, count * 8, cudaMemcpyDeviceToDevice, s) == cudaSuccess) ? 0 : 1;
    return nccl().AllGather(send, recv, count, ncclDouble, c, s) == ncclSuccess ? 0 : 1;
  }
};

// ---- loopback group: nranks contexts on one device, one host thread per rank ----
struct LoopGroup {
  int n;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  std::vector<const double*> p_lo, p_hi, p_all;  // published device pointers
  std::vector<std::vector<double>> host;          // host slots for reductions
  explicit LoopGroup(int nr) : n(nr), p_lo(nr), p_hi(nr), p_all(nr), host(nr) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

// Every copy runs on the rank's own stream and is waited for before the next barrier: a plain
// cudaMemcpy runs on the legacy stream, which does not order against the non-blocking streams the
// contexts run on, and a device-to-device (or pageable host-to-device) cudaMemcpy may return
// before the copy lands -- the peer could then overwrite its send buffer, or this rank's next
// kernel read the receive buffer, while the copy is still in flight.
struct LoopComm : psp_comm {
  std::shared_ptr<LoopGroup> g;
  int allreduce(double* d, size_t count, int op, cudaStream_t s) override {
    if (cudaStreamSynchronize(s) != cudaSuccess) return 1;
    g->host[rank].resize(count);
    if (cudaMemcpyAsync(g->host[rank].data(), d, count * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return 1;
    g->barrier();
    std::vector<double> r(g->host[0]);
    for (int q = 1; q < nranks; ++q)  // rank order: identical on every rank
      for (size_t i = 0; i < count; ++i) {
        const double v = g->host[q][i];
        r[i] = op == 0 ? r[i] + v : (op == 1 ? (v > r[i] ? v : r[i]) : (v < r[i] ? v : r[i]));
      }
    g->barrier();
    return (cudaMemcpyAsync(d, r.data(), count * 8, cudaMemcpyHostToDevice, s) == cudaSuccess &&
            cudaStreamSynchronize(s) == cudaSuccess) ? 0 : 1;
  }
  int sendrecv(const double* send_lo, double* recv_lo, size_t n_lo, const double* send_hi,
               double* recv_hi, size_t n_hi, cudaStream_t s) override {
    if (cudaStreamSynchronize(s) != cudaSuccess) return 1;
    g->p_lo[rank] = send_lo;
    g->p_hi[rank] = send_hi;
    g->barrier();
    int err = 0;
    if (rank > 0 && n_lo &&
        cudaMemcpyAsync(recv_lo, g->p_hi[rank - 1], n_lo * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess) err = 1;
    if (rank < nranks - 1 && n_hi &&
        cudaMemcpyAsync(recv_hi, g->p_lo[rank + 1], n_hi * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess) err = 1;
    if (cudaStreamSynchronize(s) != cudaSuccess) err = 1;
    g->barrier();
    return err;
  }
  int allgather(const double* send, double* recv, size_t count, cudaStream_t s) override {
    if (cudaStreamSynchronize(s) != cudaSuccess) return 1;
    g->p_all[rank] = send;
    g->barrier();
    int err = 0;
    for (int q = 0; q < nranks; ++q)
      if (cudaMemcpyAsync(recv + q * count, g->p_all[q], count * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess) err = 1;
    if (cudaStreamSynchronize(s) != cudaSuccess) err = 1;
    g->barrier();
    return err;
  }
};

// ---- process-level host transport: the caller's collective callbacks on host buffers ----
// (one process per rank, any transport the caller has -- e.g. torch.distributed over gloo; the
// tests run two processes on one GPU this way, host-mediated so no kernel waits on another rank)
struct HostComm : psp_comm {
  psp_host_transport t{};
  double* hb = nullptr;                     // pinned staging, grown on demand
  size_t cap = 0;
  ~HostComm() override {
    if (hb) cudaFreeHost(hb);
  }
  double* stage(size_t count) {
    if (count > cap) {
      if (hb) cudaFreeHost(hb);
      hb = nullptr;
      cap = 0;
      if (cudaMallocHost((void**)&hb, count * 8) != cudaSuccess) return nullptr;
      cap = count;
    }
    return hb;
  }
  int d2h(double* h, const double* d, size_t count, cudaStream_t s) {
    return (count == 0 || (cudaMemcpyAsync(h, d, count * 8, cudaMemcpyDeviceToHost, s) == cudaSuccess &&
                           cudaStreamSynchronize(s) == cudaSuccess)) ? 0 : 1;
  }
  int h2d(double* d, const double* h, size_t count, cudaStream_t s) {
    return (count == 0 || (cudaMemcpyAsync(d, h, count * 8, cudaMemcpyHostToDevice, s) == cudaSuccess &&
                           cudaStreamSynchronize(s) == cudaSuccess)) ? 0 : 1;
  }
  int allreduce(double* d, size_t count, int op, cudaStream_t s) override {
    double* h = stage(count);
    if (!h || cudaStreamSynchronize(s) != cudaSuccess || d2h(h, d, count, s)) return 1;
    if (t.allreduce(t.user, h, count, op)) return 1;
    return h2d(d, h, count, s);
  }
  int sendrecv(const double* send_lo, double* recv_lo, size_t n_lo, const double* send_hi,
               double* recv_hi, size_t n_hi, cudaStream_t s) override {
    const bool lo = rank > 0 && n_lo, hi = rank < nranks - 1 && n_hi;
    double* h = stage(2 * (n_lo + n_hi) + 1);
    if (!h || cudaStreamSynchronize(s) != cudaSuccess) return 1;
    double *sl = h, *rl = h + n_lo, *sh = h + 2 * n_lo, *rh = h + 2 * n_lo + n_hi;
    if ((lo && d2h(sl, send_lo, n_lo, s)) || (hi && d2h(sh, send_hi, n_hi, s))) return 1;
    if (t.sendrecv(t.user, lo ? sl : nullptr, lo ? rl : nullptr, lo ? n_lo : 0, hi ? sh : nullptr,
                   hi ? rh : nullptr, hi ? n_hi : 0))
      return 1;
    if ((lo && h2d(recv_lo, rl, n_lo, s)) || (hi && h2d(recv_hi, rh, n_hi, s))) return 1;
    return 0;
  }
  int allgather(const double* send, double* recv, size_t count, cudaStream_t s) override {
    double* h = stage(count * (nranks + 1));
    if (!h || cudaStreamSynchronize(s) != cudaSuccess || d2h(h, send, count, s)) return 1;
    if (t.allgather(t.user, h, h + count, count)) return 1;
    return h2d(recv, h + count, count * nranks, s);
  }
};

}  // namespace

extern "C" {

psp_status psp_comm_host_create(const psp_host_transport* t, int nranks, int rank, psp_comm** out) {
  if (!t || !out || nranks < 1 || rank < 0 || rank >= nranks || !t->allreduce || !t->sendrecv || !t->allgather)
    return PSP_E_ARG;
  auto* c = new HostComm();
  c->t = *t;
  c->nranks = nranks;
  c->rank = rank;
  *out = c;
  return PSP_OK;
}

psp_status psp_comm_unique_id(void* id) {
  if (!id) return PSP_E_ARG;
  ncclUniqueId u;
  if (!nccl().ok || nccl().GetUniqueId(&u) != ncclSuccess) return PSP_E_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id, &u, sizeof(u));
  return PSP_OK;
}

psp_status psp_comm_init(const void* id, int nranks, int rank, psp_comm** out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks) return PSP_E_ARG;
  auto* c = new NcclComm();
  c->nranks = nranks;
  c->rank = rank;
  if (nranks > 1 || id) {                          // (one rank with an id: a real NCCL comm)
    if (!id) {
      delete c;
      return PSP_E_ARG;
    }
    ncclUniqueId u;
    memcpy(&u, id, sizeof(u));
    if (!nccl().ok || nccl().CommInitRank(&c->c, nranks, u, rank) != ncclSuccess) {
      delete c;
      return PSP_E_NCCL;
    }
  }
  *out = c;
  return PSP_OK;
}

psp_status psp_comm_selftest(psp_comm* c, void* stream) {
  if (!c) return PSP_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int R = c->nranks, r = c->rank;
  constexpr int K = 8;                             // values a collective
  // device layout: [sum K | max K | min K | gather src K | gather dst R K | send lo K | send hi K |
  //                 recv lo K | recv hi K]
  const size_t total = (size_t)K * (8 + R);
  double* d = nullptr;
  if (cudaMalloc(&d, total * 8) != cudaSuccess) return PSP_E_CUDA;
  std::vector<double> h(total, -1.0);
  for (int i = 0; i < K; ++i) {
    h[i] = r + 0.5 * i;                            // sum over ranks: R(R-1)/2 + R i/2
    h[K + i] = (double)((r + i) % R) + 10.0 * i;   // a permutation over ranks: max R-1 + 10 i
    h[2 * K + i] = -(double)((r + 2 * i) % R) + 10.0 * i;   // min -(R-1) + 10 i
    h[3 * K + i] = 1000.0 * r + i;                 // gathered block q: 1000 q + i
    h[(size_t)(4 + R) * K + i] = 100.0 * r + i;     // to rank r-1 (its "hi" neighbour)
    h[(size_t)(5 + R) * K + i] = 100.0 * r + 50.0 + i;   // to rank r+1
  }
  auto fail = [&](const char* what) {
    cudaFree(d);
    return what ? (psp_status)PSP_E_NCCL : (psp_status)PSP_E_CUDA;
  };
  if (cudaMemcpyAsync(d, h.data(), total * 8, cudaMemcpyHostToDevice, s) != cudaSuccess) return fail(nullptr);
  double* dlo = d + (size_t)(6 + R) * K;
  double* dhi = d + (size_t)(7 + R) * K;
  if (c->allreduce(d, K, 0, s) || c->allreduce(d + K, K, 1, s) || c->allreduce(d + 2 * K, K, 2, s))
    return fail("allreduce");
  if (c->allgather(d + 3 * K, d + 4 * K, K, s)) return fail("allgather");
  if (c->sendrecv(d + (size_t)(4 + R) * K, dlo, K, d + (size_t)(5 + R) * K, dhi, K, s)) return fail("sendrecv");
  std::vector<double> o(total);
  if (cudaMemcpyAsync(o.data(), d, total * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return fail(nullptr);
  cudaFree(d);
  bool ok = true;
  for (int i = 0; i < K; ++i) {
    ok = ok && o[i] == 0.5 * R * (R - 1) + 0.5 * R * i;
    ok = ok && o[K + i] == (R - 1) + 10.0 * i;
    ok = ok && o[2 * K + i] == -(double)(R - 1) + 10.0 * i;
    for (int q = 0; q < R; ++q) ok = ok && o[(size_t)(4 + q) * K + i] == 1000.0 * q + i;
    if (r > 0) ok = ok && o[(size_t)(6 + R) * K + i] == 100.0 * (r - 1) + 50.0 + i;   // rank r-1's hi
    else ok = ok && o[(size_t)(6 + R) * K + i] == -1.0;                             // untouched
    if (r < R - 1) ok = ok && o[(size_t)(7 + R) * K + i] == 100.0 * (r + 1) + i;    // rank r+1's lo
    else ok = ok && o[(size_t)(7 + R) * K + i] == -1.0;
  }
  return ok ? PSP_OK : PSP_E_NCCL;
}

psp_status psp_comm_loopback_create(int nranks, psp_comm** out) {
  if (!out || nranks < 1) return PSP_E_ARG;
  auto g = std::make_shared<LoopGroup>(nranks);
  for (int r = 0; r < nranks; ++r) {
    auto* c = new LoopComm();
    c->nranks = nranks;
    c->rank = r;
    c->g = g;
    out[r] = c;
  }
  return PSP_OK;
}

psp_status psp_comm_destroy(psp_comm* c) {
  delete c;
  return PSP_OK;
}

}  // extern "C"
