// Direct-to-peer transport over CUDA IPC peer memory ("the a2a buffers drive the
// peak", "we only need buffers for 2 heads").
//
// Every rank owns a symmetric region (cudaMalloc, same layout on every rank) that holds the layer's
// whole workspace -- so each receive buffer sits at the same offset on every rank -- plus
// synchronisation flags and the dW all-reduce scratch. Peers map it with cudaIpcOpenMemHandle (NVLink 5
// / NVSwitch on a B200 box; the same device in the multi-process tests). Data moves by PUSH: a rank
// writes its block straight into the owner's receive buffer -- with the copy engines for the generic
// collectives here, and from the producing kernels' epilogues on the fused paths (the projection GEMM's
// TMA stores, the attention epilogue, the dQ conversion; layer.cpp) -- so no send buffer and no NCCL
// SMs are involved.
//
// Ordering is carried by 32-bit flags in the receiver's region, written and waited on by the GPU front
// end (cuStreamWriteValue32 / cuStreamWaitValue32, no SM spins), per collective epoch e (every rank
// issues the same sequence of collectives, so epochs agree):
//   ready[e % 64][p] = e   peer p's stream has reached collective e: its receive buffers may be written
//   done [e % 64][p] = e   peer p has pushed all its data of collective e into this rank's buffers
// The default WriteValue32 is preceded by a memory fence, so a done flag is seen only after the pushed
// data. Slots are per epoch (not one flag per peer) because the overlapped schedule runs collectives on
// two streams, whose progress is not ordered.
#include <cuda.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>

#include "kernels.h"
#include "upipe_internal.h"

namespace upipe {

namespace {

using PFN_streamValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct MemOps {
  PFN_streamValue32 write = nullptr, wait = nullptr;
};

const MemOps& memops() {
  static const MemOps m = [] {
    MemOps r;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      r.write = reinterpret_cast<PFN_streamValue32>(p);
    p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      r.wait = reinterpret_cast<PFN_streamValue32>(p);
    return r;
  }();
  return m;
}

__global__ void ipc_sum_kernel(const float* const* bufs, int C, size_t begin, size_t end, float* dst, float* mirror) {
  for (size_t i = begin + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < end; i += (size_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int p = 0; p < C; ++p) s += bufs[p][i];   // fixed rank order: deterministic
    dst[i] = s;
    mirror[i] = s;
  }
}

}  // namespace

size_t ipc_region_bytes(size_t ws_bytes, size_t scratch_bytes) {
  return kIpcFlagBytes + ((ws_bytes + 255) & ~size_t(255)) + scratch_bytes;
}

class IpcTransport final : public Transport {
 public:
  IpcTransport(int C, int rank, int dev, void* base, size_t bytes, size_t ws_bytes)
      : C_(C), rank_(rank), dev_(dev), base_(static_cast<char*>(base)), bytes_(bytes), ws_bytes_(ws_bytes) {
    peer_.assign(C, nullptr);
    peer_[rank] = base_;
  }
  ~IpcTransport() override {
    for (int p = 0; p < C_; ++p)
      if (p != rank_ && peer_[p]) cudaIpcCloseMemHandle(peer_[p]);
    if (dev_ptrs_) cudaFree(dev_ptrs_);
    if (base_) cudaFree(base_);
  }
  int size() const override { return C_; }
  int rank() const override { return rank_; }
  int kind() const override { return 3; }
  int device() const override { return dev_; }
  char* workspace() override { return base_ + kIpcFlagBytes; }
  size_t workspace_bytes() const override { return ws_bytes_; }
  bool peer_capable() const override { return connected_; }
  void* peer_ptr(int p, const void* local) const override {
    const char* l = static_cast<const char*>(local);
    if (l < base_ || l >= base_ + bytes_ || !peer_[p]) return nullptr;
    return peer_[p] + (l - base_);
  }

  upipe_status_t connect(const uint8_t* handles, std::string& err) {
    for (int p = 0; p < C_; ++p) {
      if (p == rank_) continue;
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + (size_t)p * UPIPE_IPC_HANDLE_BYTES, sizeof h);
      void* ptr = nullptr;
      cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        err = std::string("cudaIpcOpenMemHandle(peer ") + std::to_string(p) + "): " + cudaGetErrorString(e);
        return UPIPE_ERR_COMM;
      }
      peer_[p] = static_cast<char*>(ptr);
    }
    if (!memops().write || !memops().wait) {
      err = "cuStreamWriteValue32 / cuStreamWaitValue32 entry points unavailable";
      return UPIPE_ERR_COMM;
    }
    connected_ = true;
    return UPIPE_OK;
  }

  // ---- flag protocol (epoch e, slot e % kIpcSlots)
  uint32_t next_epoch() override { return ++epoch_; }
  upipe_status_t signal_ready(uint32_t e, int first, int n, cudaStream_t s, std::string& err) override {
    for (int p = first; p < first + n; ++p)
      if (p != rank_ && !write_flag(p, kReady, e, s, err)) return UPIPE_ERR_COMM;
    return UPIPE_OK;
  }
  upipe_status_t wait_ready(uint32_t e, int p, cudaStream_t s, std::string& err) override {
    return wait_flag(kReady, e, p, s, err) ? UPIPE_OK : UPIPE_ERR_COMM;
  }
  upipe_status_t signal_done(uint32_t e, int p, cudaStream_t s, std::string& err) override {
    return write_flag(p, kDone, e, s, err) ? UPIPE_OK : UPIPE_ERR_COMM;
  }
  upipe_status_t wait_done(uint32_t e, int first, int n, cudaStream_t s, std::string& err) override {
    for (int p = first; p < first + n; ++p)
      if (p != rank_ && !wait_flag(kDone, e, p, s, err)) return UPIPE_ERR_COMM;
    return UPIPE_OK;
  }
  // push handshake around a producer that writes into every group peer's receive buffers
  upipe_status_t push_begin(int first, int n, cudaStream_t s, uint32_t* epoch, std::string& err) override {
    const uint32_t e = next_epoch();
    *epoch = e;
    if (upipe_status_t st = signal_ready(e, first, n, s, err)) return st;
    for (int p = first; p < first + n; ++p)
      if (p != rank_)
        if (upipe_status_t st = wait_ready(e, p, s, err)) return st;
    return UPIPE_OK;
  }
  upipe_status_t push_end(uint32_t e, int first, int n, cudaStream_t s, std::string& err) override {
    for (int p = first; p < first + n; ++p)
      if (p != rank_)
        if (upipe_status_t st = signal_done(e, p, s, err)) return st;
    return wait_done(e, first, n, s, err);
  }

  // ---- generic collectives by copy-engine push into the owners' receive buffers
  upipe_status_t alltoall_group(const void* send, void* recv, size_t bytes, int first, int n, cudaStream_t s,
                                std::string& err) override {
    uint32_t e = 0;
    if (upipe_status_t st = push_begin(first, n, s, &e, err)) return st;
    for (int i = 0; i < n; ++i) {
      const int p = first + (rank_ - first + i) % n;    // start with self, then the next ranks (spread the load)
      char* dst = static_cast<char*>(p == rank_ ? recv : peer_ptr(p, recv));
      if (!dst) {
        err = "IPC all-to-all: receive buffer outside the symmetric region";
        return UPIPE_ERR_INVALID_ARG;
      }
      cudaError_t ce = cudaMemcpyAsync(dst + (size_t)(rank_ - first) * bytes,
                                       static_cast<const char*>(send) + (size_t)(p - first) * bytes, bytes,
                                       cudaMemcpyDeviceToDevice, s);
      if (ce != cudaSuccess) {
        err = std::string("IPC all-to-all copy: ") + cudaGetErrorString(ce);
        return UPIPE_ERR_CUDA;
      }
    }
    return push_end(e, first, n, s, err);
  }

  upipe_status_t sendrecv(const void* send, int dst, void* recv, int src, size_t bytes, cudaStream_t s,
                          std::string& err) override {
    const uint32_t e = next_epoch();
    if (src != rank_ && !write_flag(src, kReady, e, s, err)) return UPIPE_ERR_COMM;   // my recv is free
    if (dst == rank_) {
      if (cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess) {
        err = "IPC sendrecv: local copy";
        return UPIPE_ERR_CUDA;
      }
      return UPIPE_OK;
    }
    if (!wait_flag(kReady, e, dst, s, err)) return UPIPE_ERR_COMM;
    void* d = peer_ptr(dst, recv);
    if (!d) {
      err = "IPC sendrecv: receive buffer outside the symmetric region";
      return UPIPE_ERR_INVALID_ARG;
    }
    if (cudaMemcpyAsync(d, send, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess) {
      err = "IPC sendrecv: peer copy";
      return UPIPE_ERR_CUDA;
    }
    if (!write_flag(dst, kDone, e, s, err)) return UPIPE_ERR_COMM;
    return wait_flag(kDone, e, src, s, err) ? UPIPE_OK : UPIPE_ERR_COMM;
  }

  // dW all-reduce: stage into the symmetric scratch, barrier, every rank sums its slice over all peers'
  // scratch (NVLink reads, fixed rank order) into its dW and its scratch, barrier, copy the other slices
  // from their owners, barrier (scratch free for the next call).
  upipe_status_t allreduce_sum_f32(float* buf, size_t n, cudaStream_t s, std::string& err) override {
    const size_t scratch_bytes = bytes_ - kIpcFlagBytes - ((ws_bytes_ + 255) & ~size_t(255));
    if (n * 4 > scratch_bytes) {
      err = "IPC all-reduce: scratch too small";
      return UPIPE_ERR_WORKSPACE;
    }
    float* scratch = reinterpret_cast<float*>(base_ + kIpcFlagBytes + ((ws_bytes_ + 255) & ~size_t(255)));
    if (cudaMemcpyAsync(scratch, buf, n * 4, cudaMemcpyDeviceToDevice, s) != cudaSuccess) {
      err = "IPC all-reduce: stage";
      return UPIPE_ERR_CUDA;
    }
    if (upipe_status_t st = barrier(s, err)) return st;
    if (!dev_ptrs_ && cudaMalloc(&dev_ptrs_, sizeof(float*) * 64) != cudaSuccess) {
      err = "IPC all-reduce: cudaMalloc";
      return UPIPE_ERR_CUDA;
    }
    std::vector<const float*> h(C_);
    for (int p = 0; p < C_; ++p) h[p] = static_cast<const float*>(peer_ptr(p, scratch));
    cudaMemcpyAsync(dev_ptrs_, h.data(), sizeof(float*) * C_, cudaMemcpyHostToDevice, s);
    const size_t chunk = (n + C_ - 1) / C_;
    const size_t b = std::min(n, chunk * rank_), en = std::min(n, chunk * (rank_ + 1));
    if (en > b) {
      ipc_sum_kernel<<<148 * 4, 256, 0, s>>>(dev_ptrs_, C_, b, en, buf, scratch);
      count_launches(1);
    }
    if (upipe_status_t st = barrier(s, err)) return st;
    for (int p = 0; p < C_; ++p) {
      if (p == rank_) continue;
      const size_t pb = std::min(n, chunk * p), pe = std::min(n, chunk * (p + 1));
      if (pe > pb)
        cudaMemcpyAsync(buf + pb, static_cast<const float*>(peer_ptr(p, scratch)) + pb, (pe - pb) * 4,
                        cudaMemcpyDeviceToDevice, s);
    }
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) {
      err = std::string("IPC all-reduce: ") + cudaGetErrorString(ce);
      return UPIPE_ERR_CUDA;
    }
    return barrier(s, err);
  }

 private:
  enum { kReady = 0, kDone = 1 };
  upipe_status_t barrier(cudaStream_t s, std::string& err) {
    const uint32_t e = next_epoch();
    for (int p = 0; p < C_; ++p)
      if (p != rank_ && !write_flag(p, kDone, e, s, err)) return UPIPE_ERR_COMM;
    return wait_done(e, 0, C_, s, err);
  }
  // flag word of (kind, slot of e, source rank src) inside a region
  static size_t flag_off(int kind, uint32_t e, int src) {
    return ((size_t)kind * kIpcSlots + e % kIpcSlots) * 64 * 4 + (size_t)src * 4;
  }
  bool write_flag(int p, int kind, uint32_t e, cudaStream_t s, std::string& err) {
    const CUdeviceptr a = reinterpret_cast<CUdeviceptr>(peer_[p] + flag_off(kind, e, rank_));
    const CUresult r = memops().write(reinterpret_cast<CUstream>(s), a, e, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) {
      err = "cuStreamWriteValue32 failed (" + std::to_string((int)r) + ")";
      return false;
    }
    return true;
  }
  bool wait_flag(int kind, uint32_t e, int src, cudaStream_t s, std::string& err) {
    const CUdeviceptr a = reinterpret_cast<CUdeviceptr>(base_ + flag_off(kind, e, src));
    const CUresult r = memops().wait(reinterpret_cast<CUstream>(s), a, e, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) {
      err = "cuStreamWaitValue32 failed (" + std::to_string((int)r) + ")";
      return false;
    }
    return true;
  }
  int C_, rank_, dev_;
  char* base_;
  size_t bytes_, ws_bytes_;
  std::vector<char*> peer_;
  bool connected_ = false;
  uint32_t epoch_ = 0;
  float** dev_ptrs_ = nullptr;
};

std::unique_ptr<Transport> make_ipc_transport(int C, int rank, int device, size_t ws_bytes, size_t scratch_bytes,
                                              uint8_t* handle_out, std::string& err) {
  const size_t bytes = ipc_region_bytes(ws_bytes, scratch_bytes);
  void* base = nullptr;
  cudaError_t e = cudaMalloc(&base, bytes);
  if (e != cudaSuccess) {
    err = std::string("IPC region cudaMalloc: ") + cudaGetErrorString(e);
    return nullptr;
  }
  if ((e = cudaMemset(base, 0, kIpcFlagBytes)) != cudaSuccess) {   // flags start at epoch 0
    cudaFree(base);
    err = std::string("IPC flags memset: ") + cudaGetErrorString(e);
    return nullptr;
  }
  cudaIpcMemHandle_t h;
  if ((e = cudaIpcGetMemHandle(&h, base)) != cudaSuccess) {
    cudaFree(base);
    err = std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e);
    return nullptr;
  }
  static_assert(sizeof(cudaIpcMemHandle_t) <= UPIPE_IPC_HANDLE_BYTES, "IPC handle size");
  std::memset(handle_out, 0, UPIPE_IPC_HANDLE_BYTES);
  std::memcpy(handle_out, &h, sizeof h);
  return std::make_unique<IpcTransport>(C, rank, device, base, bytes, ws_bytes);
}

upipe_status_t ipc_connect(Transport* t, const uint8_t* handles, std::string& err) {
  auto* it = dynamic_cast<IpcTransport*>(t);
  if (!it) {
    err = "ctx was not created with upipe_ipc_create";
    return UPIPE_ERR_STATE;
  }
  return it->connect(handles, err);
}

}  // namespace upipe
