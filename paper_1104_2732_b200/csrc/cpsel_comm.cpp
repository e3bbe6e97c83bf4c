#include "cpsel_comm.h"

#include <chrono>
#include <cstdlib>

namespace cpsel {

bool LoopGroup::barrier(double timeout_s) {
  std::unique_lock<std::mutex> l(mu);
  if (broken) return false;
  const unsigned long long g0 = gen;
  if (++arrived == world) {
    arrived = 0;
    ++gen;
    cv.notify_all();
    return true;
  }
  const bool ok = cv.wait_for(l, std::chrono::duration<double>(timeout_s), [&] { return gen != g0 || broken; });
  if (gen != g0) return true;
  if (!ok) {
    broken = true;
    cv.notify_all();
  }
  return false;
}

static const char* cuda_msg(cudaError_t e) { return e == cudaSuccess ? nullptr : cudaGetErrorString(e); }

const char* Comm::allgatherv(const void* send, void* out, const size_t* bytes, cudaStream_t st) {
  char* o = static_cast<char*>(out);
  if (nccl) {
    const NcclApi& nc = nccl_api();
    bool equal = true;
    for (int q = 1; q < world; ++q) equal &= bytes[q] == bytes[0];
    ncclResult_t r;
    if (equal) {
      if (bytes[0] == 0) return nullptr;
      r = nc.AllGather(send, out, bytes[0], ncclUint8, nccl, st);
      return r == ncclSuccess ? nullptr : nc.GetErrorString(r);
    }
    // all-gather-v as grouped broadcasts (rank q is the root of block q)
    if ((r = nc.GroupStart()) != ncclSuccess) return nc.GetErrorString(r);
    size_t off = 0;
    for (int q = 0; q < world; ++q) {
      if (bytes[q]) {
        r = nc.Broadcast(q == rank ? send : nullptr, o + off, bytes[q], ncclUint8, q, nccl, st);
        if (r != ncclSuccess) {
          nc.GroupEnd();
          return nc.GetErrorString(r);
        }
      }
      off += bytes[q];
    }
    r = nc.GroupEnd();
    return r == ncclSuccess ? nullptr : nc.GetErrorString(r);
  }
  if (!loop) return "no communicator";
  LoopGroup& g = *loop;
  const char* m;
  if ((m = cuda_msg(cudaEventRecord(ev_ready, st)))) return m;
  {
    std::lock_guard<std::mutex> l(g.mu);
    g.src[rank] = send;
  }
  if (!g.barrier(timeout_s)) return "loopback collective: a peer rank did not arrive (timeout)";
  size_t off = 0;
  for (int q = 0; q < world; ++q) {
    if (bytes[q] && (o + off) != g.src[q]) {
      if (q != rank && (m = cuda_msg(cudaStreamWaitEvent(st, g.ready[q], 0)))) return m;
      if ((m = cuda_msg(cudaMemcpyAsync(o + off, g.src[q], bytes[q], cudaMemcpyDeviceToDevice, st)))) return m;
    }
    off += bytes[q];
  }
  if ((m = cuda_msg(cudaEventRecord(ev_done, st)))) return m;
  if (!g.barrier(timeout_s)) return "loopback collective: a peer rank did not arrive (timeout)";
  // no rank may overwrite its send buffer before every peer's copies of it are done
  for (int q = 0; q < world; ++q)
    if (q != rank && (m = cuda_msg(cudaStreamWaitEvent(st, g.done[q], 0)))) return m;
  return nullptr;
}

const char* Comm::allgather(const void* send, void* out, size_t bytes, cudaStream_t st) {
  std::vector<size_t> b(world, bytes);
  return allgatherv(send, out, b.data(), st);
}

const char* Comm::attach_loop(std::shared_ptr<LoopGroup> g, int r) {
  release();
  if (!g || r < 0 || r >= g->world) return "bad loopback group / rank";
  cudaError_t e;
  if ((e = cudaEventCreateWithFlags(&ev_ready, cudaEventDisableTiming)) != cudaSuccess) return cudaGetErrorString(e);
  if ((e = cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming)) != cudaSuccess) return cudaGetErrorString(e);
  {
    std::lock_guard<std::mutex> l(g->mu);
    if (g->attached[r]) return "loopback rank already attached";
    g->attached[r] = 1;
    g->ready[r] = ev_ready;
    g->done[r] = ev_done;
  }
  loop = std::move(g);
  rank = r;
  world = loop->world;
  return nullptr;
}

const char* Comm::health() const {
  if (nccl) {
    const NcclApi& nc = nccl_api();
    if (!nc.CommGetAsyncError) return nullptr;
    ncclResult_t a = ncclSuccess;
    const ncclResult_t r = nc.CommGetAsyncError(nccl, &a);
    if (r != ncclSuccess) return nc.GetErrorString(r);
    if (a != ncclSuccess && a != ncclInProgress) return nc.GetErrorString(a);
    return nullptr;
  }
  if (loop) {
    std::lock_guard<std::mutex> l(loop->mu);
    if (loop->broken) return "loopback group broken (a peer rank timed out)";
  }
  return nullptr;
}

void Comm::abort() {
  if (nccl && nccl_api().ok) {
    if (nccl_api().CommAbort) nccl_api().CommAbort(nccl);
    nccl = nullptr;  // never CommDestroy an aborted communicator
  }
  if (loop) {
    std::lock_guard<std::mutex> l(loop->mu);
    loop->broken = true;  // the peers' next (or current) barrier fails instead of hanging
    loop->cv.notify_all();
  }
  release();
}

double comm_timeout_from_env(double dflt) {
  const char* e = getenv("CPSEL_COMM_TIMEOUT_S");
  if (!e) return dflt;
  const double v = atof(e);
  return v > 0 ? v : dflt;
}

void Comm::release() {
  if (nccl && nccl_api().ok) nccl_api().CommDestroy(nccl);
  nccl = nullptr;
  if (loop) {
    std::lock_guard<std::mutex> l(loop->mu);
    loop->attached[rank] = 0;
    loop->ready[rank] = nullptr;
    loop->done[rank] = nullptr;
  }
  loop.reset();
  if (ev_ready) cudaEventDestroy(ev_ready);
  if (ev_done) cudaEventDestroy(ev_done);
  ev_ready = ev_done = nullptr;
  rank = 0;
  world = 1;
}

}  // namespace cpsel
