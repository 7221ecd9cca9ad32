// Collectives of the UPipe path.
//
//  * SelfTransport   C = 1: the all-to-alls are identities (A20: no a2a at C = 1).
//  * NcclTransport   one process per GPU; equal-block all-to-all as one grouped
//                    ncclSend/ncclRecv per peer over NVLink 5 / NVSwitch; fp32
//                    all-reduce of dW.
//  * FabricTransport C ranks as host threads of one process (each with its own
//                    stream): peers' send buffers are read with device-to-device
//                    copies ordered by CUDA events and host barriers. Runs the
//                    sharded path (C = 2..8) on a single GPU for parity tests.
#include <nccl.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>

#include "upipe_internal.h"

namespace upipe {

// Default failure detection: poll the stream until it drains or the timeout passes.
upipe_status_t Transport::wait(cudaStream_t s, double timeout_s, std::string& err) {
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return UPIPE_OK;
    if (q != cudaErrorNotReady) {
      err = std::string("stream: ") + cudaGetErrorString(q);
      return UPIPE_ERR_CUDA;
    }
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (timeout_s > 0 && el > timeout_s) {
      err = "timeout waiting for the stream";
      return UPIPE_ERR_COMM;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
}

namespace {

class SelfTransport final : public Transport {
 public:
  int size() const override { return 1; }
  int rank() const override { return 0; }
  int kind() const override { return 0; }
  upipe_status_t alltoall_group(const void* send, void* recv, size_t bytes, int, int, cudaStream_t s,
                                std::string& err) override {
    return copy(send, recv, bytes, s, err);
  }
  upipe_status_t sendrecv(const void* send, int, void* recv, int, size_t bytes, cudaStream_t s, std::string& err) override {
    return copy(send, recv, bytes, s, err);
  }
  upipe_status_t allreduce_sum_f32(float*, size_t, cudaStream_t, std::string&) override { return UPIPE_OK; }

 private:
  static upipe_status_t copy(const void* send, void* recv, size_t bytes, cudaStream_t s, std::string& err) {
    if (send == recv || bytes == 0) return UPIPE_OK;
    cudaError_t e = cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) {
      err = cudaGetErrorString(e);
      return UPIPE_ERR_CUDA;
    }
    return UPIPE_OK;
  }
};

class NcclTransport final : public Transport {
 public:
  NcclTransport(ncclComm_t c, int C, int r, int max_ctas, int dev)
      : comm_(c), C_(C), rank_(r), max_ctas_(max_ctas), dev_(dev) {}
  ~NcclTransport() override {
    if (comm_) {
      if (aborted_) return;                      // ncclCommAbort already released it
      ncclCommDestroy(comm_);
    }
  }
  int size() const override { return C_; }
  int rank() const override { return rank_; }
  int kind() const override { return 1; }
  int max_ctas() const override { return max_ctas_; }
  int device() const override { return dev_; }
  // Watchdog (SURVEY §5 failure detection): ncclCommGetAsyncError is polled while the stream drains;
  // an asynchronous error (e.g. a peer's network/process failure) or a timeout aborts the communicator,
  // which makes this rank's pending NCCL kernels return, so the rank fails instead of hanging.
  upipe_status_t wait(cudaStream_t s, double timeout_s, std::string& err) override {
    if (aborted_) {
      err = "communicator was aborted";
      return UPIPE_ERR_COMM;
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      ncclResult_t ae = ncclSuccess;
      ncclResult_t r = ncclCommGetAsyncError(comm_, &ae);
      if (r != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress)) {
        err = std::string("NCCL asynchronous error: ") + ncclGetErrorString(r != ncclSuccess ? r : ae);
        abort_comm();
        return UPIPE_ERR_COMM;
      }
      const cudaError_t q = cudaStreamQuery(s);
      if (q == cudaSuccess) return UPIPE_OK;
      if (q != cudaErrorNotReady) {
        err = std::string("stream: ") + cudaGetErrorString(q);
        return UPIPE_ERR_CUDA;
      }
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (timeout_s > 0 && el > timeout_s) {
        char m[160];
        snprintf(m, sizeof m, "rank %d: no progress for %.1f s (a peer failed or stalled); communicator aborted",
                 rank_, el);
        err = m;
        abort_comm();
        return UPIPE_ERR_COMM;
      }
      std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
  }
  upipe_status_t alltoall_group(const void* send, void* recv, size_t bytes, int first, int n, cudaStream_t s,
                                std::string& err) override {
    ncclResult_t r = ncclGroupStart();
    for (int p = 0; p < n && r == ncclSuccess; ++p) {
      r = ncclSend(static_cast<const char*>(send) + p * bytes, bytes, ncclUint8, first + p, comm_, s);
      if (r == ncclSuccess) r = ncclRecv(static_cast<char*>(recv) + p * bytes, bytes, ncclUint8, first + p, comm_, s);
    }
    ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess) {
      err = std::string("NCCL all-to-all: ") + ncclGetErrorString(r != ncclSuccess ? r : r2);
      return UPIPE_ERR_COMM;
    }
    return UPIPE_OK;
  }
  upipe_status_t sendrecv(const void* send, int dst, void* recv, int src, size_t bytes, cudaStream_t s,
                          std::string& err) override {
    ncclResult_t r = ncclGroupStart();
    if (r == ncclSuccess) r = ncclSend(send, bytes, ncclUint8, dst, comm_, s);
    if (r == ncclSuccess) r = ncclRecv(recv, bytes, ncclUint8, src, comm_, s);
    ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess) {
      err = std::string("NCCL ring send/recv: ") + ncclGetErrorString(r != ncclSuccess ? r : r2);
      return UPIPE_ERR_COMM;
    }
    return UPIPE_OK;
  }
  upipe_status_t allreduce_sum_f32(float* buf, size_t n, cudaStream_t s, std::string& err) override {
    ncclResult_t r = ncclAllReduce(buf, buf, n, ncclFloat32, ncclSum, comm_, s);
    if (r != ncclSuccess) {
      err = std::string("NCCL all-reduce: ") + ncclGetErrorString(r);
      return UPIPE_ERR_COMM;
    }
    return UPIPE_OK;
  }

 private:
  void abort_comm() {
    if (!aborted_ && comm_) ncclCommAbort(comm_);
    aborted_ = true;
  }
  ncclComm_t comm_;
  int C_, rank_, max_ctas_, dev_;
  bool aborted_ = false;
};

}  // namespace

}  // namespace upipe

// ------------------------------------------------------------------ fabric (single process, C threads)
struct upipe_fabric_s {
  int C = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<const void*> ptr;
  std::vector<cudaEvent_t> ev_a, ev_b;
  std::vector<int> device;

  // Host barrier across the C ranks; false on timeout (a peer failed or never called).
  bool barrier(int timeout_s = 120) {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t gen = generation;
    if (++arrived == C) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return true;
    }
    return cv.wait_for(lk, std::chrono::seconds(timeout_s), [&] { return generation != gen; });
  }
};

namespace upipe {
namespace {

__global__ void fabric_sum_kernel(float* const* bufs, int C, size_t begin, size_t end, float* dst) {
  for (size_t i = begin + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < end; i += (size_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int p = 0; p < C; ++p) s += bufs[p][i];
    dst[i] = s;
  }
}

class FabricTransport final : public Transport {
 public:
  FabricTransport(upipe_fabric_t f, int r) : f_(f), rank_(r) {}
  ~FabricTransport() override {
    if (dev_ptrs_) cudaFree(dev_ptrs_);
  }
  int size() const override { return f_->C; }
  int rank() const override { return rank_; }
  int kind() const override { return 2; }
  int device() const override { return f_->device[rank_]; }

  upipe_status_t alltoall_group(const void* send, void* recv, size_t bytes, int first, int n, cudaStream_t s,
                                std::string& err) override {
    if (!sync_publish(send, s, err)) return UPIPE_ERR_COMM;
    for (int p = 0; p < n; ++p) {
      const int peer = first + p;
      if (peer != rank_) cudaStreamWaitEvent(s, f_->ev_a[peer], 0);
      const char* src = static_cast<const char*>(f_->ptr[peer]) + (size_t)(rank_ - first) * bytes;
      cudaError_t e = cudaMemcpyAsync(static_cast<char*>(recv) + (size_t)p * bytes, src, bytes,
                                      cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) {
        err = cudaGetErrorString(e);
        return UPIPE_ERR_CUDA;
      }
    }
    return finish(s, err) ? UPIPE_OK : UPIPE_ERR_COMM;
  }

  upipe_status_t sendrecv(const void* send, int dst, void* recv, int src, size_t bytes, cudaStream_t s,
                          std::string& err) override {
    (void)dst;                                    // the receiver pulls: rank dst reads our published buffer
    if (!sync_publish(send, s, err)) return UPIPE_ERR_COMM;
    if (src != rank_) cudaStreamWaitEvent(s, f_->ev_a[src], 0);
    cudaError_t e = cudaMemcpyAsync(recv, f_->ptr[src], bytes, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) {
      err = cudaGetErrorString(e);
      return UPIPE_ERR_CUDA;
    }
    return finish(s, err) ? UPIPE_OK : UPIPE_ERR_COMM;
  }

  upipe_status_t allreduce_sum_f32(float* buf, size_t n, cudaStream_t s, std::string& err) override {
    const int C = f_->C;
    if (!sync_publish(buf, s, err)) return UPIPE_ERR_COMM;
    for (int p = 0; p < C; ++p)
      if (p != rank_) cudaStreamWaitEvent(s, f_->ev_a[p], 0);
    if (!dev_ptrs_ && cudaMalloc(&dev_ptrs_, sizeof(float*) * 64) != cudaSuccess) {
      err = "fabric: cudaMalloc";
      return UPIPE_ERR_CUDA;
    }
    std::vector<float*> h(C);
    for (int p = 0; p < C; ++p) h[p] = const_cast<float*>(static_cast<const float*>(f_->ptr[p]));
    cudaMemcpyAsync(dev_ptrs_, h.data(), sizeof(float*) * C, cudaMemcpyHostToDevice, s);
    const size_t chunk = (n + C - 1) / C;
    const size_t b = std::min(n, chunk * rank_), e = std::min(n, chunk * (rank_ + 1));
    if (e > b) {
      fabric_sum_kernel<<<148 * 4, 256, 0, s>>>(dev_ptrs_, C, b, e, buf);
      count_launches(1);
    }
    // everyone's owned slice is reduced; then copy the other slices from their owners
    if (!sync_publish(buf, s, err)) return UPIPE_ERR_COMM;
    for (int p = 0; p < C; ++p) {
      if (p == rank_) continue;
      cudaStreamWaitEvent(s, f_->ev_a[p], 0);
      const size_t pb = std::min(n, chunk * p), pe = std::min(n, chunk * (p + 1));
      if (pe > pb)
        cudaMemcpyAsync(buf + pb, static_cast<const float*>(f_->ptr[p]) + pb, (pe - pb) * 4, cudaMemcpyDeviceToDevice, s);
    }
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) {
      err = cudaGetErrorString(ce);
      return UPIPE_ERR_CUDA;
    }
    return finish(s, err) ? UPIPE_OK : UPIPE_ERR_COMM;
  }

 private:
  // Record "my buffer is ready" and publish its pointer; returns after all ranks did the same.
  bool sync_publish(const void* p, cudaStream_t s, std::string& err) {
    cudaEventRecord(f_->ev_a[rank_], s);
    f_->ptr[rank_] = p;
    if (!f_->barrier()) {
      err = "fabric barrier timeout (a peer rank failed or never entered the collective)";
      return false;
    }
    return true;
  }
  // Record "done reading peers" and make my stream wait until all peers finished reading my buffer.
  bool finish(cudaStream_t s, std::string& err) {
    cudaEventRecord(f_->ev_b[rank_], s);
    if (!f_->barrier()) {
      err = "fabric barrier timeout";
      return false;
    }
    for (int p = 0; p < f_->C; ++p)
      if (p != rank_) cudaStreamWaitEvent(s, f_->ev_b[p], 0);
    if (!f_->barrier()) {
      err = "fabric barrier timeout";
      return false;
    }
    return true;
  }
  upipe_fabric_t f_;
  int rank_;
  float** dev_ptrs_ = nullptr;
};

}  // namespace

std::unique_ptr<Transport> make_self_transport() { return std::make_unique<SelfTransport>(); }

std::unique_ptr<Transport> make_nccl_transport(const uint8_t* uid, int C, int rank, std::string& err) {
  ncclUniqueId id;
  static_assert(sizeof(ncclUniqueId) <= UPIPE_UID_BYTES, "uid size");
  std::memcpy(&id, uid, sizeof(id));
  // CTA cap: the all-to-all of the next chunk runs while the attention kernels hold
  // one CTA per SM with all of its shared memory, so NCCL's CTAs cannot share SMs with them; an
  // uncapped communicator could park many CTAs on SMs while it waits for a late peer. NVLink 5 needs
  // only a few channels per peer for these message sizes (MBs), so cap them (UPIPE_NCCL_MAX_CTAS,
  // default 16 of 148 SMs).
  int max_ctas = 16;
  if (const char* e = getenv("UPIPE_NCCL_MAX_CTAS")) max_ctas = atoi(e) > 0 ? atoi(e) : max_ctas;
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.blocking = 1;
  cfg.maxCTAs = max_ctas;
  cfg.minCTAs = max_ctas < 4 ? max_ctas : 4;
  cfg.commName = "upipe";
  ncclComm_t comm = nullptr;
  ncclResult_t r = ncclCommInitRankConfig(&comm, C, id, rank, &cfg);
  if (r != ncclSuccess) {
    err = std::string("ncclCommInitRankConfig: ") + ncclGetErrorString(r);
    return nullptr;
  }
  int n = 0, me = -1, dev = -1, ver = 0;
  ncclCommCount(comm, &n);
  ncclCommUserRank(comm, &me);
  ncclCommCuDevice(comm, &dev);
  ncclGetVersion(&ver);
  if (!(getenv("UPIPE_QUIET") && getenv("UPIPE_QUIET")[0] == '1'))
    fprintf(stderr, "[upipe] NCCL %d communicator: rank %d of %d on cuda:%d, max CTAs %d\n", ver, me, n, dev, max_ctas);
  if (n != C || me != rank) {
    err = "NCCL communicator does not match (cp_size, cp_rank)";
    ncclCommDestroy(comm);
    return nullptr;
  }
  return std::make_unique<NcclTransport>(comm, C, rank, max_ctas, dev);
}

std::unique_ptr<Transport> make_fabric_transport(upipe_fabric_t f, int rank, int device, std::string& err) {
  if (!f || rank < 0 || rank >= f->C) {
    err = "fabric: bad rank";
    return nullptr;
  }
  {
    std::lock_guard<std::mutex> lk(f->mu);
    if (cudaEventCreateWithFlags(&f->ev_a[rank], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&f->ev_b[rank], cudaEventDisableTiming) != cudaSuccess) {
      err = "fabric: cudaEventCreate failed";
      return nullptr;
    }
    f->device[rank] = device;
  }
  return std::make_unique<FabricTransport>(f, rank);
}

}  // namespace upipe

extern "C" upipe_status_t upipe_fabric_create(upipe_fabric_t* fabric, int cp_size) {
  if (!fabric || cp_size < 1 || cp_size > 64) return UPIPE_ERR_INVALID_ARG;
  auto* f = new upipe_fabric_s();
  f->C = cp_size;
  f->ptr.assign(cp_size, nullptr);
  f->ev_a.assign(cp_size, nullptr);
  f->ev_b.assign(cp_size, nullptr);
  f->device.assign(cp_size, 0);
  *fabric = f;
  return UPIPE_OK;
}

extern "C" upipe_status_t upipe_fabric_destroy(upipe_fabric_t f) {
  if (!f) return UPIPE_ERR_INVALID_ARG;
  for (int p = 0; p < f->C; ++p) {
    if (f->ev_a[p]) cudaEventDestroy(f->ev_a[p]);
    if (f->ev_b[p]) cudaEventDestroy(f->ev_b[p]);
  }
  delete f;
  return UPIPE_OK;
}
