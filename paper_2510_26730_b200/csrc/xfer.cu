// xfer.cu — the physical transfer engine behind the C ABI (ef_xfer_*):
// expert copies from pinned host memory into HBM, issued in the reference's
// TransferQueue order (memory.py:184-202: MISS before PREFETCH, FIFO within a
// class; simcore.h TransferQueue) on a dedicated high-priority copy stream,
// at most `max_inflight` outstanding (1 = the reference's single serial link,
// engine.py:328-354), each bracketed by CUDA events so completion can be
// polled, waited on from the host or from another stream, and its measured
// rate folded into a BandwidthEstimator (memory.py:205-236, alpha 0.25).
//
// The decode engine (engine.cu) drives its own copies from the scheduler's
// logical clock; this engine is the standalone form of the same machinery
// for a caller that runs its own scheduler.
#include <cuda_runtime.h>

#include <algorithm>
#include <deque>
#include <memory>
#include <vector>

#include "capi_util.h"

using namespace ef;

namespace {
struct XferReq {
  const void* src;
  void* dst;
  int64_t bytes;
};
struct Inflight {
  int64_t ticket;
  cudaEvent_t a, b;
  int64_t bytes;
};
}  // namespace

struct ef_xfer {
  int device = 0, max_inflight = 1;
  cudaStream_t stream = nullptr;
  TransferQueue q;
  std::vector<XferReq> reqs;  // by ticket
  std::vector<char> done;     // by ticket
  std::deque<Inflight> inflight;
  std::vector<cudaEvent_t> pool;
  std::vector<int64_t> completed;  // since the last poll
  BandwidthEstimator bw{false, 0.0, 0.25};
  int64_t n_completed = 0;

  cudaEvent_t take() {
    cudaEvent_t e;
    if (!pool.empty()) {
      e = pool.back();
      pool.pop_back();
      return e;
    }
    if (cudaEventCreate(&e) != cudaSuccess) throw CudaErr("cudaEventCreate failed");
    return e;
  }
  void reap() {
    while (!inflight.empty()) {
      Inflight& f = inflight.front();
      const cudaError_t r = cudaEventQuery(f.b);
      if (r == cudaErrorNotReady) break;
      if (r != cudaSuccess) throw CudaErr(std::string("copy failed: ") + cudaGetErrorString(r));
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, f.a, f.b) == cudaSuccess && ms > 0.f)
        bw.observe(f.bytes, (int64_t)(ms * 1e6));
      done[f.ticket] = 1;
      completed.push_back(f.ticket);
      ++n_completed;
      pool.push_back(f.a);
      pool.push_back(f.b);
      inflight.pop_front();
    }
  }
  int pump() {
    reap();
    int issued = 0;
    TransferRequest r;
    while ((int)inflight.size() < max_inflight && q.next(&r)) {
      const int64_t t = (int64_t)r.key;
      const XferReq& rq = reqs[t];
      Inflight f{t, take(), take(), rq.bytes};
      if (cudaEventRecord(f.a, stream) != cudaSuccess ||
          cudaMemcpyAsync(rq.dst, rq.src, rq.bytes, cudaMemcpyHostToDevice, stream) != cudaSuccess ||
          cudaEventRecord(f.b, stream) != cudaSuccess)
        throw CudaErr("could not issue the copy");
      inflight.push_back(f);
      ++issued;
    }
    return issued;
  }
  ~ef_xfer() {
    if (stream) cudaStreamSynchronize(stream);
    for (auto& f : inflight) {
      cudaEventDestroy(f.a);
      cudaEventDestroy(f.b);
    }
    for (auto e : pool) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
  }
};

extern "C" int ef_xfer_create(int32_t device, int32_t max_inflight, ef_xfer** out) {
  EF_TRY({
    if (max_inflight < 1) throw ValueError("max_inflight must be >= 1");
    auto x = std::make_unique<ef_xfer>();
    x->device = device;
    x->max_inflight = max_inflight;
    if (cudaSetDevice(device) != cudaSuccess) throw CudaErr("cudaSetDevice failed");
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&x->stream, cudaStreamNonBlocking, hi) != cudaSuccess)
      throw CudaErr("could not create the copy stream");
    *out = x.release();
  });
}

extern "C" void ef_xfer_destroy(ef_xfer* x) { delete x; }

extern "C" int ef_xfer_submit(ef_xfer* x, int32_t layer, int32_t expert, int32_t priority,
                              const void* src, void* dst, int64_t bytes, int64_t* ticket) {
  (void)layer;
  (void)expert;
  EF_TRY({
    if (priority < 0 || priority > 1) throw ValueError("priority must be 0 (MISS) or 1 (PREFETCH)");
    if (!src || !dst || bytes <= 0) throw ValueError("bad copy arguments");
    const int64_t t = (int64_t)x->reqs.size();
    x->reqs.push_back(XferReq{src, dst, bytes});
    x->done.push_back(0);
    x->q.enqueue((uint64_t)t, priority);
    *ticket = t;
  });
}

extern "C" int ef_xfer_pump(ef_xfer* x, int32_t* issued) {
  EF_TRY({
    const int n = x->pump();
    if (issued) *issued = n;
  });
}

extern "C" int ef_xfer_poll(ef_xfer* x, int64_t* tickets, int32_t max, int32_t* n) {
  EF_TRY({
    x->pump();
    const int m = std::min<int>((int)x->completed.size(), std::max(0, max));
    for (int i = 0; i < m; ++i) tickets[i] = x->completed[i];
    x->completed.erase(x->completed.begin(), x->completed.begin() + m);
    *n = m;
  });
}

extern "C" int ef_xfer_wait(ef_xfer* x, int64_t ticket) {
  EF_TRY({
    if (ticket < 0 || ticket >= (int64_t)x->reqs.size()) throw ValueError("unknown ticket");
    for (;;) {
      x->pump();
      if (x->done[ticket]) return EF_OK;
      if (x->inflight.empty()) throw RuntimeErr("ticket is neither queued nor in flight");
      if (cudaEventSynchronize(x->inflight.front().b) != cudaSuccess)
        throw CudaErr("cudaEventSynchronize failed");
    }
  });
}

extern "C" int ef_xfer_stream_wait(ef_xfer* x, int64_t ticket, void* stream) {
  EF_TRY({
    if (ticket < 0 || ticket >= (int64_t)x->reqs.size()) throw ValueError("unknown ticket");
    x->pump();
    if (x->done[ticket]) return EF_OK;
    for (const Inflight& f : x->inflight)
      if (f.ticket == ticket) {
        if (cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), f.b, 0) != cudaSuccess)
          throw CudaErr("cudaStreamWaitEvent failed");
        return EF_OK;
      }
    throw RuntimeErr("ticket not issued yet (pump first, or raise max_inflight)");
  });
}

extern "C" int ef_xfer_bandwidth(ef_xfer* x, double* bytes_per_s, int64_t* completed) {
  EF_TRY({
    x->reap();
    *bytes_per_s = x->n_completed ? x->bw.estimate() : 0.0;
    *completed = x->n_completed;
  });
}
