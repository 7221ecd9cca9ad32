// Internal host-side structures of libupipe (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/upipe.h"

namespace upipe {

// ------------------------------------------------------------------ plan (DESIGN A8)
struct Plan {
  int C = 1;                  // Ulysses degree: ranks of one all-to-all group (= cp_size unless ring > 1)
  int ring = 1;               // ring degree r of the UPipe x Ring hybrid (DESIGN A27); cp_size = C * ring
  upipe_shape_t sh{};
  int64_t S_l = 0, S = 0;
  int R = 1, qpd = 1, kv_res = 1, sigma = 1, nstages = 1;
  int d = 0, Hq = 0, Hkv = 0, D = 0, U = 0;

  // GQA schedule, closed form: stage s = (super-stage b, position r); device p holds KV heads
  // [(b*C + p)*kv_res, +kv_res) and q heads [kv0*R + r*qpd, +qpd).
  int kv0(int s, int p) const { return ((s / sigma) * C + p) * kv_res; }
  int q0(int s, int p) const { return kv0(s, p) * R + (s % sigma) * qpd; }
  // naive (UPIPE_FLAG_NAIVE_KV): every stage re-projects and re-sends the K/V heads its
  // queries read, and sends their gradients back at once (no super-stage reuse)
  bool naive = false;
  bool kv_sent(int s) const { return naive || (s % sigma) == 0; }
  bool kv_last(int s) const { return naive || (s % sigma) == sigma - 1; }
  int kv_group(int s) const { return naive ? s : s / sigma; }   // stages sharing one K/V receive buffer
  int kv_pos(int s) const { return naive ? 0 : s % sigma; }     // position within that group
  // backward dX through the pre-allocated gradient buffer G [S_l][(Hq + 2 Hkv) d] bf16 (DESIGN A30) instead of
  // a fp32 accumulator [S_l][D]: with more than one stage, not naive, and only where G is no larger
  bool gbuf() const { return !naive && nstages > 1 && (int64_t)(Hq + 2 * Hkv) * d * 2 <= (int64_t)D * 4; }
  // per-device step of the first q head / kv head between consecutive devices (same for every s)
  int q_dev_stride() const { return kv_res * R; }
  int kv_dev_stride() const { return kv_res; }
};

// Returns UPIPE_OK or the status of the first violated precondition, with msg naming it.
upipe_status_t validate_shape(int C, const upipe_shape_t* sh, std::string& msg);
Plan make_plan(int C, const upipe_shape_t& sh);

// Workspace layout: byte offsets into the caller's workspace for one pass.
// [2] = the two buffer sets of the overlapped (pipelined) schedule; in the sequential
// schedule (or C == 1) index 1 aliases index 0.
struct FwdWs {
  size_t qsend[2], qrecv[2], ksend, krecv[2], vsend, vrecv[2], osend[2], orecv[2];
  size_t kring[2], vring[2], oacc, opart, lsepart;   // ring hybrid only
  size_t total;
};
struct BwdWs {
  size_t qsend[2], qrecv[2], ksend, krecv[2], vsend, vrecv[2], dosend[2], dorecv[2], dsend[2], drecv[2], dqacc[2],
      dqsend[2], dqrecv[2], dkacc, dvacc, dksend, dvsend, dkrecv, dvrecv, dxacc;
  size_t gbuf;                                        // pre-allocated gradient buffer (not with naive KV)
  size_t dqsem;                                       // UPIPE_FLAG_DETERMINISTIC dQ-order semaphores (int32)
  size_t qn[2], kn[2], dgam;                          // Qwen3 q/k norm (shape.qk_norm_eps > 0) only
  size_t kring[2], vring[2], dkring[2], dvring[2];   // ring hybrid only
  size_t total;
};
// direct: UPIPE_FLAG_DIRECT layout (receive buffers only; the send offsets alias them and are unused)
FwdWs fwd_workspace(const Plan& p, bool overlap, bool direct = false);
BwdWs bwd_workspace(const Plan& p, bool overlap, bool direct = false);

// ------------------------------------------------------------------ transport
class Transport {
 public:
  virtual ~Transport() = default;
  virtual int size() const = 0;
  virtual int rank() const = 0;
  // Equal-block all-to-all: block p of `send` (bytes at send + p*bytes) goes to rank p, which stores
  // it as block `rank()` of its `recv`. send and recv must not overlap (except C == 1).
  upipe_status_t alltoall(const void* send, void* recv, size_t bytes, cudaStream_t s, std::string& err) {
    return alltoall_group(send, recv, bytes, 0, size(), s, err);
  }
  // The same inside the group of ranks [first, first + n) (a Ulysses group of the ring hybrid):
  // block p goes to rank first + p, which stores it as block rank() - first.
  virtual upipe_status_t alltoall_group(const void* send, void* recv, size_t bytes, int first, int n, cudaStream_t s,
                                        std::string& err) = 0;
  // Ring step: `bytes` of `send` go to rank dst while `bytes` from rank src land in `recv` (every
  // rank calls it together; send and recv must not overlap).
  virtual upipe_status_t sendrecv(const void* send, int dst, void* recv, int src, size_t bytes, cudaStream_t s,
                                  std::string& err) = 0;
  virtual upipe_status_t allreduce_sum_f32(float* buf, size_t n, cudaStream_t s, std::string& err) = 0;
  // Failure detection (upipe_wait): wait for `s` while checking the transport for asynchronous errors;
  // on an error or after timeout_s (<= 0: none) the transport aborts its communicator (so this rank's
  // collectives return instead of waiting for a dead peer forever) and reports UPIPE_ERR_COMM.
  virtual upipe_status_t wait(cudaStream_t s, double timeout_s, std::string& err);
  virtual int kind() const = 0;          // upipe_comm_info_t.transport
  virtual int max_ctas() const { return 0; }
  virtual int device() const { return -1; }

  // ---- direct-to-peer (IpcTransport in ipc.cu). A transport with peer memory owns the
  // layer's workspace (a symmetric region: every buffer at the same offset on every rank) and lets
  // producers write straight into the owners' receive buffers between push_begin and push_end.
  virtual char* workspace() { return nullptr; }            // non-null: the layer's workspace lives here
  virtual size_t workspace_bytes() const { return 0; }
  virtual bool peer_capable() const { return false; }
  virtual void* peer_ptr(int p, const void* local) const { (void)p; (void)local; return nullptr; }
  virtual uint32_t next_epoch() { return 0; }
  virtual upipe_status_t signal_ready(uint32_t, int, int, cudaStream_t, std::string& err) { err = "no peer memory"; return UPIPE_ERR_STATE; }
  virtual upipe_status_t wait_ready(uint32_t, int, cudaStream_t, std::string& err) { err = "no peer memory"; return UPIPE_ERR_STATE; }
  virtual upipe_status_t signal_done(uint32_t, int, cudaStream_t, std::string& err) { err = "no peer memory"; return UPIPE_ERR_STATE; }
  virtual upipe_status_t wait_done(uint32_t, int, int, cudaStream_t, std::string& err) { err = "no peer memory"; return UPIPE_ERR_STATE; }
  // all group peers have reached this collective (their receive buffers are free) ...
  virtual upipe_status_t push_begin(int, int, cudaStream_t, uint32_t*, std::string& err) { err = "no peer memory"; return UPIPE_ERR_STATE; }
  // ... this rank's pushes are complete (signalled to each peer) and every peer's pushes have landed here
  virtual upipe_status_t push_end(uint32_t, int, int, cudaStream_t, std::string& err) { err = "no peer memory"; return UPIPE_ERR_STATE; }
};

constexpr size_t kIpcFlagBytes = 64 * 1024;   // ready / done flags: 2 x 64 epoch slots x 64 ranks x 4 B
constexpr uint32_t kIpcSlots = 64;
size_t ipc_region_bytes(size_t ws_bytes, size_t scratch_bytes);
std::unique_ptr<Transport> make_ipc_transport(int C, int rank, int device, size_t ws_bytes, size_t scratch_bytes,
                                              uint8_t* handle_out, std::string& err);
upipe_status_t ipc_connect(Transport* t, const uint8_t* handles, std::string& err);

std::unique_ptr<Transport> make_self_transport();
std::unique_ptr<Transport> make_nccl_transport(const uint8_t* uid, int C, int rank, std::string& err);
std::unique_ptr<Transport> make_fabric_transport(upipe_fabric_t f, int rank, int device, std::string& err);

// Event-bracketed timing of layer steps (upipe_set_trace / upipe_trace_read).
struct Tracer {
  bool on = false;
  struct Rec {
    int cat;
    cudaEvent_t a, b;
    const char* label;   // static string naming the step ("out proj", "dX(dQ)", ...)
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
  ~Tracer() {
    for (auto& r : recs) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

void count_launches(uint64_t n);

}  // namespace upipe

namespace upipe {
// Streams and events of the overlapped schedule (comm stream = high priority, owned by the ctx).
struct Pipe {
  cudaStream_t comm = nullptr;
  static constexpr int kEvents = 24;
  cudaEvent_t ev[kEvents] = {};
  bool ready = false;
  ~Pipe() {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    if (comm) cudaStreamDestroy(comm);
  }
};

}  // namespace upipe

namespace upipe {
// Overlapped UPipe schedule (double-buffered chunk set, next stage's all-to-all on the comm stream).
// The ring hybrid runs its Ulysses all-to-alls sequentially on the compute stream; its ring transfers
// are issued on the ctx's comm stream one step ahead of the attention (layer.cpp).
// Direct-to-peer mode (UPIPE_FLAG_DIRECT): producers write into the owners' receive buffers;
// one buffer set, no send buffers, no comm stream.
inline bool direct_enabled(uint32_t flags, const Plan& P) {
  return (flags & UPIPE_FLAG_DIRECT) && P.C > 1;
}
inline bool overlap_enabled(uint32_t flags, const Plan& P) {
  return P.C > 1 && P.ring == 1 && !(flags & UPIPE_FLAG_SYNC_COMM) && !direct_enabled(flags, P);
}
}  // namespace upipe

namespace upipe {
// RoPE rotation tables owned by the ctx (RopeRef in kernels.h), rebuilt when (base, d) change or a
// longer sequence arrives. A few MB at most (hi: S/1024 x d/2, lo: 1024 x d/2 float2).
struct RopeTables {
  float base = 0.f;
  int d = 0;
  int64_t n_hi = 0;
  float2* hi = nullptr;
  float2* lo = nullptr;
  ~RopeTables() {
    if (hi) cudaFree(hi);
    if (lo) cudaFree(lo);
  }
};
}  // namespace upipe

struct upipe_ctx_s {
  upipe_probe_t probe{-1, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                      nullptr, nullptr, nullptr};   // test-only layout probe (upipe_test_set_probe)
  upipe::RopeTables rope;
  upipe::Pipe pipe;
  upipe::Tracer tracer;
  int device = 0;
  int C = 1, rank = 0;
  uint32_t flags = 0;
  std::unique_ptr<upipe::Transport> transport;
  std::string last_error;
  bool alive = true;
  bool ipc_pending = false;   // upipe_ipc_create done, upipe_ipc_connect not yet
};
