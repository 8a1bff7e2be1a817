// mock_nccl.cpp -- TEST ONLY: an in-process stand-in for the handful of NCCL entry points the
// library uses (include/zz.h multi-GPU path), so that the collective zz_tgevc runs with
// several ranks -- one host thread each, all on the same GPU -- inside one test process.
// NCCL itself refuses two ranks on one device; this transport copies device buffers between
// the ranks' streams with cudaMemcpyAsync and orders them with events, after a host-side
// rendezvous per operation.  Loaded by the library instead of libnccl when ZZ_NCCL_LIB names
// it (tests/test_gpu.py::test_multirank_collective_mock).
#include <cuda_runtime.h>
#include <nccl.h>
#include <string.h>

#include <condition_variable>
#include <map>
#include <mutex>
#include <string>
#include <vector>

namespace {

struct Post {              // one side of a transfer, published by its owner
  const void* ptr = nullptr;
  size_t bytes = 0;
  cudaEvent_t ready = nullptr;   // the data is in place on the owner's stream
  bool posted = false;
  cudaEvent_t done = nullptr;    // the consumer's copy has been enqueued after this event
  bool consumed = false;
};

struct World {
  int n = 0, joined = 0;
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::string, Post> posts;   // key: op sequence + roles
  std::vector<long> seq;               // per-rank sequence number of collective ops
};

std::mutex g_mu;
std::map<std::string, World*> g_worlds;

struct Comm {
  World* w;
  int rank;
  // pending operations of an open group
  struct Op { bool send; const void* sbuf; void* rbuf; size_t bytes; int peer; cudaStream_t st; };
  std::vector<Op> group;
  int group_depth = 0;
};

thread_local std::vector<Comm*> t_open;   // comms with an open group on this thread

size_t esize(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
  }
}

std::string key(long s, int from, int to) { return std::to_string(s) + ":" + std::to_string(from) + ">" + std::to_string(to); }

// publish `ptr` (ready after the work queued on `st`) for `to`
void publish(World* w, const std::string& k, const void* ptr, size_t bytes, cudaStream_t st) {
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  cudaEventRecord(ev, st);
  std::unique_lock<std::mutex> lk(w->mu);
  Post& p = w->posts[k];
  p.ptr = ptr; p.bytes = bytes; p.ready = ev; p.posted = true;
  w->cv.notify_all();
}
// copy the data published under `k` into `dst` on `st`; tell the publisher when it may reuse
void consume(World* w, const std::string& k, void* dst, size_t bytes, cudaStream_t st) {
  std::unique_lock<std::mutex> lk(w->mu);
  w->cv.wait(lk, [&] { return w->posts[k].posted; });
  Post& p = w->posts[k];
  lk.unlock();
  cudaStreamWaitEvent(st, p.ready, 0);
  if (dst != p.ptr && bytes) cudaMemcpyAsync(dst, p.ptr, bytes, cudaMemcpyDeviceToDevice, st);
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  cudaEventRecord(ev, st);
  lk.lock();
  p.done = ev; p.consumed = true;
  w->cv.notify_all();
}
// the publisher's stream waits until the consumer's copy is done
void await_consumed(World* w, const std::string& k, cudaStream_t st) {
  std::unique_lock<std::mutex> lk(w->mu);
  w->cv.wait(lk, [&] { return w->posts[k].consumed; });
  cudaEvent_t d = w->posts[k].done;
  lk.unlock();
  cudaStreamWaitEvent(st, d, 0);
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  static std::mutex m;
  static long counter = 0;
  std::lock_guard<std::mutex> lk(m);
  memset(id->internal, 0, sizeof(id->internal));
  snprintf(id->internal, sizeof(id->internal), "mock-%ld", ++counter);
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  World* w;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    std::string k(id.internal);
    if (!g_worlds.count(k)) { g_worlds[k] = new World(); g_worlds[k]->n = nranks; g_worlds[k]->seq.assign(nranks, 0); }
    w = g_worlds[k];
  }
  {
    std::unique_lock<std::mutex> lk(w->mu);
    w->joined++;
    w->cv.notify_all();
    w->cv.wait(lk, [&] { return w->joined >= w->n; });
  }
  Comm* c = new Comm();
  c->w = w;
  c->rank = rank;
  *comm = reinterpret_cast<ncclComm_t>(c);
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  delete reinterpret_cast<Comm*>(comm);
  return ncclSuccess;
}

ncclResult_t ncclBroadcast(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t dt, int root,
                           ncclComm_t comm, cudaStream_t st) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  World* w = c->w;
  const long s = w->seq[c->rank]++;
  const size_t bytes = count * esize(dt);
  if (c->rank == root) {
    if (recvbuff != sendbuff) cudaMemcpyAsync(recvbuff, sendbuff, bytes, cudaMemcpyDeviceToDevice, st);
    for (int q = 0; q < w->n; ++q)
      if (q != root) publish(w, key(s, root, q), sendbuff, bytes, st);
    for (int q = 0; q < w->n; ++q)
      if (q != root) await_consumed(w, key(s, root, q), st);
  } else {
    consume(w, key(s, root, c->rank), recvbuff, bytes, st);
  }
  return ncclSuccess;
}

ncclResult_t ncclGroupStart() { return ncclSuccess; }

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm, cudaStream_t st) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  c->group.push_back(Comm::Op{true, buf, nullptr, count * esize(dt), peer, st});
  bool found = false;
  for (Comm* o : t_open) found |= (o == c);
  if (!found) t_open.push_back(c);
  return ncclSuccess;
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm, cudaStream_t st) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  c->group.push_back(Comm::Op{false, nullptr, buf, count * esize(dt), peer, st});
  bool found = false;
  for (Comm* o : t_open) found |= (o == c);
  if (!found) t_open.push_back(c);
  return ncclSuccess;
}

// a group: every send is published, then every receive consumed, then every send awaited --
// the sequence number of the group is per (sender, receiver) pair
ncclResult_t ncclGroupEnd() {
  for (Comm* c : t_open) {
    World* w = c->w;
    const long s = w->seq[c->rank]++;
    std::vector<std::string> sent;
    for (auto& op : c->group)
      if (op.send) {
        const std::string k = "g" + key(s, c->rank, op.peer);
        publish(w, k, op.sbuf, op.bytes, op.st);
        sent.push_back(k);
      }
    for (auto& op : c->group)
      if (!op.send) consume(w, "g" + key(s, op.peer, c->rank), op.rbuf, op.bytes, op.st);
    size_t i = 0;
    for (auto& op : c->group)
      if (op.send) await_consumed(w, sent[i++], op.st);
    c->group.clear();
  }
  t_open.clear();
  return ncclSuccess;
}

}  // extern "C"
