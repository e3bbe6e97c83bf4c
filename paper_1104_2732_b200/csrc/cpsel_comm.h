// Collectives of the sharded path (a6, "partial sums from several GPUs are added"): the
// all-gather of the per-rank tuples / sample shares and the all-gather-v of the bracket contents.
// Two transports behind one interface:
//  * NCCL over the ranks' communicator (one process per GPU, NVLink/NVSwitch);
//  * a loopback group: G virtual ranks of ONE process on one device, each a host thread with its
//    own cpsel ctx and stream (SURVEY §4 "G virtual shards on one GPU").  A collective is two host
//    barriers around device-to-device copies; stream order is carried across ranks by CUDA events
//    (each rank's copies wait for every source's "ready" event, and every rank waits for all
//    ranks' "done" events before it may overwrite its own send buffer).
// The sharded driver code above this interface is the same for both.
#pragma once
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <memory>
#include <mutex>
#include <vector>

#include "cpsel_nccl.h"

namespace cpsel {

struct LoopGroup {
  explicit LoopGroup(int w) : world(w), src(w, nullptr), ready(w, nullptr), done(w, nullptr), attached(w, 0) {}
  const int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  bool broken = false;  // a rank timed out: every later barrier fails at once
  std::vector<const void*> src;
  std::vector<cudaEvent_t> ready, done;  // owned by the attached ranks' Comm
  std::vector<int> attached;
  // all `world` ranks arrive; false on timeout (the group is then broken)
  bool barrier(double timeout_s);
};

struct Comm {
  ncclComm_t nccl = nullptr;
  std::shared_ptr<LoopGroup> loop;
  int rank = 0, world = 1;
  cudaEvent_t ev_ready = nullptr, ev_done = nullptr;  // loopback: this rank's events
  double timeout_s = 120.0;  // a collective that has not completed after this long fails the call


  bool active() const { return nccl != nullptr || loop != nullptr; }
  // out <- the concatenation over ranks q of (q's send, bytes[q]) (bytes[] the same on every rank;
  // send may alias this rank's block of out).  Returns nullptr or an error message.
  const char* allgatherv(const void* send, void* out, const size_t* bytes, cudaStream_t st);
  // equal sizes: out <- concat of every rank's `bytes` bytes
  const char* allgather(const void* send, void* out, size_t bytes, cudaStream_t st);
  // attach to a loopback group as `rank` (creates the events); nullptr or an error message
  const char* attach_loop(std::shared_ptr<LoopGroup> g, int rank);
  void release();  // destroy the communicator / detach from the group
  // failure detection while a host waits on a collective: nullptr while healthy, else a message
  // (an NCCL asynchronous error, e.g. a peer process that died; a broken loopback group)
  const char* health() const;
  // tear the communicator down without waiting for peers (after health() or a timeout failed);
  // the ctx must be re-initialised with cpsel_comm_init* before the next sharded call
  void abort();
};

// CPSEL_COMM_TIMEOUT_S (seconds, > 0) overrides Comm::timeout_s at comm init
double comm_timeout_from_env(double dflt);

}  // namespace cpsel
