// hjb_comm.h -- the exchange steps of the slab-decomposed path: halo rows between
// neighbouring slabs and all-gathers of small per-rank values (Krylov dot products, nonlinear
// residual, changed counts) and of coarse multigrid rows at the gather level.
//
// Two backends behind one interface:
//   NcclComm   -- production: one process per GPU, NCCL point-to-point (grouped ncclSend/ncclRecv)
//                 for halos and ncclAllGather for reductions, all on the grid's stream (NVLink /
//                 NVSwitch between B200s).
//   ThreadComm -- TEST-ONLY: several ranks as host threads of ONE process on one device, halos by
//                 cudaMemcpyAsync between the ranks' buffers.  Ordering uses CUDA events
//                 (cudaStreamWaitEvent) plus host barriers; no kernel ever waits on another rank's
//                 kernel.  It exists so the decomposition logic (partition, halos, gather level,
//                 deterministic reductions) runs on the one GPU a test box has.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace hjb {

struct Msg {
  int peer;
  const void* send;
  void* recv;
  size_t bytes;
};

struct Comm {
  int rank = 0, nranks = 1;
  virtual ~Comm() {}
  // every message: send `bytes` at send to peer, receive `bytes` from peer into recv
  virtual cudaError_t exchange(cudaStream_t st, const Msg* m, int nm, std::string* err) = 0;
  // recv[q * bytes ...] = send of rank q, for every q (rank order)
  virtual cudaError_t allgather(cudaStream_t st, const void* send, void* recv, size_t bytes, std::string* err) = 0;
};

// ------------------------------------------------------------------------------------ NCCL
struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  static bool init(NcclComm* c, const void* id, int rank, int nranks, std::string* err) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclResult_t r = ncclCommInitRank(&c->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
      *err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
      return false;
    }
    c->rank = rank;
    c->nranks = nranks;
    return true;
  }
  ~NcclComm() override {
    if (comm) ncclCommDestroy(comm);
  }
  cudaError_t exchange(cudaStream_t st, const Msg* m, int nm, std::string* err) override {
    ncclResult_t r = ncclGroupStart();
    for (int i = 0; i < nm && r == ncclSuccess; ++i) {
      r = ncclSend(m[i].send, m[i].bytes, ncclChar, m[i].peer, comm, st);
      if (r == ncclSuccess) r = ncclRecv(m[i].recv, m[i].bytes, ncclChar, m[i].peer, comm, st);
    }
    ncclResult_t r2 = ncclGroupEnd();
    if (r == ncclSuccess) r = r2;
    if (r != ncclSuccess) {
      *err = std::string("nccl halo exchange: ") + ncclGetErrorString(r);
      return cudaErrorUnknown;
    }
    return cudaSuccess;
  }
  cudaError_t allgather(cudaStream_t st, const void* send, void* recv, size_t bytes, std::string* err) override {
    ncclResult_t r = ncclAllGather(send, recv, bytes, ncclChar, comm, st);
    if (r != ncclSuccess) {
      *err = std::string("ncclAllGather: ") + ncclGetErrorString(r);
      return cudaErrorUnknown;
    }
    return cudaSuccess;
  }
};

// ------------------------------------------------------------------------------ ThreadComm
struct ThreadGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  struct Slot {
    cudaEvent_t ready = nullptr, done = nullptr;
    std::vector<Msg> msgs;
    const void* gsend = nullptr;
  };
  std::vector<Slot> slots;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long gen = generation;
    if (++arrived == n) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

inline std::mutex& thread_registry_mu() {
  static std::mutex m;
  return m;
}
inline std::map<std::string, std::weak_ptr<ThreadGroup>>& thread_registry() {
  static std::map<std::string, std::weak_ptr<ThreadGroup>> r;
  return r;
}

struct ThreadComm : Comm {
  std::shared_ptr<ThreadGroup> grp;
  static bool init(ThreadComm* c, const void* key, int rank, int nranks, std::string* err) {
    const std::string k((const char*)key, 128);
    {
      std::lock_guard<std::mutex> lk(thread_registry_mu());
      auto& reg = thread_registry();
      auto it = reg.find(k);
      if (it != reg.end()) c->grp = it->second.lock();
      if (!c->grp) {
        c->grp = std::make_shared<ThreadGroup>();
        c->grp->n = nranks;
        c->grp->slots.resize(nranks);
        reg[k] = c->grp;
      }
    }
    if (c->grp->n != nranks) {
      *err = "thread comm: nranks differs between ranks of one group";
      return false;
    }
    c->rank = rank;
    c->nranks = nranks;
    auto& s = c->grp->slots[rank];
    if (cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming) != cudaSuccess) {
      *err = "thread comm: event create";
      return false;
    }
    c->grp->barrier();  // every rank has its events before anyone communicates
    return true;
  }
  ~ThreadComm() override {
    if (!grp) return;
    auto& s = grp->slots[rank];
    if (s.ready) cudaEventDestroy(s.ready);
    if (s.done) cudaEventDestroy(s.done);
  }
  cudaError_t exchange(cudaStream_t st, const Msg* m, int nm, std::string* err) override {
    ThreadGroup& G = *grp;
    auto& me = G.slots[rank];
    me.msgs.assign(m, m + nm);
    cudaEventRecord(me.ready, st);
    G.barrier();  // all sends published
    for (int i = 0; i < nm; ++i) {
      const auto& peer = G.slots[m[i].peer];
      const Msg* src = nullptr;
      for (const Msg& pm : peer.msgs)
        if (pm.peer == rank) src = &pm;
      if (!src || src->bytes != m[i].bytes) {
        *err = "thread comm: unmatched halo message";
        G.barrier();
        G.barrier();
        return cudaErrorInvalidValue;
      }
      cudaStreamWaitEvent(st, peer.ready, 0);
      cudaError_t e = cudaMemcpyAsync(m[i].recv, src->send, m[i].bytes, cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) { *err = cudaGetErrorString(e); }
    }
    cudaEventRecord(me.done, st);
    G.barrier();  // all copies enqueued
    for (int i = 0; i < nm; ++i) cudaStreamWaitEvent(st, G.slots[m[i].peer].done, 0);
    G.barrier();  // nobody re-records ready/done before every rank waited on them
    return cudaGetLastError();
  }
  cudaError_t allgather(cudaStream_t st, const void* send, void* recv, size_t bytes, std::string* err) override {
    ThreadGroup& G = *grp;
    auto& me = G.slots[rank];
    me.gsend = send;
    cudaEventRecord(me.ready, st);
    G.barrier();
    for (int q = 0; q < nranks; ++q) {
      cudaStreamWaitEvent(st, G.slots[q].ready, 0);
      cudaError_t e = cudaMemcpyAsync((char*)recv + (size_t)q * bytes, G.slots[q].gsend, bytes,
                                      cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) *err = cudaGetErrorString(e);
    }
    cudaEventRecord(me.done, st);
    G.barrier();
    for (int q = 0; q < nranks; ++q) cudaStreamWaitEvent(st, G.slots[q].done, 0);
    G.barrier();
    return cudaGetLastError();
  }
};

}  // namespace hjb
