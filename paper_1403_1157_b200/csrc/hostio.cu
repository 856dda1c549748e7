// tdg_apply_host: the reference call shape (apply / apply_f on host arrays,
// reference operator.py:253-288) without a pinned caller buffer.  Host data
// in any memory moves through pinned staging buffers: a pool of host
// threads copies one piece into staging while the DMA engine moves the
// previous one, and the volume kernel runs in element chunks so the
// copy-out of a chunk starts as soon as it is written.
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <unistd.h>

#include "ctx.cuh"

using namespace tdg;

namespace {

// Persistent worker pool for host memcpy (parallel first-touch page
// faults and memory bandwidth); run() splits [0, n) into one slice per
// worker plus the calling thread and returns when all are done.
class CopyPool {
 public:
  explicit CopyPool(int n) {
    for (int i = 0; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return int(th_.size()) + 1; }
  void run(const std::function<void(int, int)>& f) {
    {
      std::lock_guard<std::mutex> g(m_);
      f_ = &f;
      pending_ = int(th_.size());
      ++gen_;
    }
    cv_.notify_all();
    f(0, size());
    std::unique_lock<std::mutex> g(m_);
    done_.wait(g, [this] { return pending_ == 0; });
    f_ = nullptr;
  }

 private:
  void loop(int i) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int, int)>* f;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        f = f_;
      }
      (*f)(i + 1, size());
      std::lock_guard<std::mutex> g(m_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::function<void(int, int)>* f_ = nullptr;
  int pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// Process-wide staging (allocated on the first tdg_apply_host call, kept
// until exit; one call at a time).
constexpr int kStage = 3;
constexpr size_t kStageBytes = size_t(64) << 20;
struct Staging {
  std::mutex call;
  double* buf[kStage] = {};
  int dev = -1;
  cudaEvent_t ev[kStage] = {};
  CopyPool* pool = nullptr;
  pid_t pid = 0;  // a forked child has no pool threads (nor CUDA state)
};
Staging g_stage;

int ensure_staging() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (g_stage.pid != getpid()) {  // first call, or a fork: start afresh (the parent's are leaked)
    for (int b = 0; b < kStage; ++b) {
      g_stage.buf[b] = nullptr;
      g_stage.ev[b] = nullptr;
    }
    g_stage.pool = nullptr;
    g_stage.dev = -1;
    g_stage.pid = getpid();
  }
  if (g_stage.pool && g_stage.dev == dev) return TDG_OK;
  for (int b = 0; b < kStage; ++b) {
    if (g_stage.buf[b]) cudaFreeHost(g_stage.buf[b]);
    if (g_stage.ev[b]) cudaEventDestroy(g_stage.ev[b]);
    g_stage.buf[b] = nullptr;
    g_stage.ev[b] = nullptr;
  }
  for (int b = 0; b < kStage; ++b) {
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&g_stage.buf[b]), kStageBytes,
                                  cudaHostAllocPortable);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g_stage.ev[b], cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "tdg_apply_host: pinned staging");
  }
  g_stage.dev = dev;
  if (!g_stage.pool) {
    const unsigned hw = std::thread::hardware_concurrency();
    const int n = int(std::min(16u, std::max(hw, 2u))) - 1;
    g_stage.pool = new CopyPool(n);
  }
  return TDG_OK;
}

void par_copy(void* dst, const void* src, size_t bytes) {
  if (bytes < (size_t(4) << 20)) {
    std::memcpy(dst, src, bytes);
    return;
  }
  g_stage.pool->run([&](int i, int n) {
    const size_t a = bytes * i / n / 64 * 64, b = i + 1 == n ? bytes : bytes * (i + 1) / n / 64 * 64;
    std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
  });
}

struct Piece {
  size_t off, len;  // bytes
  int chunk;        // volume chunk that writes it (copy-out)
};

}  // namespace

extern "C" int tdg_apply_host(tdg_ctx* ctx, const double* U_host, double* R_host, double* U_dev,
                              double* R_dev, double t, int mass_inverse, void* stream) {
  (void)t;
  if (!ctx || !U_host || !R_host || !U_dev || !R_dev) return fail(TDG_E_INVALID, "null argument");
  const size_t sn = size_t(ctx->d.n_species) * ctx->d.nb;
  const int64_t ne = ctx->d.n_elements;
  const size_t ubytes = size_t(ne + ctx->d.n_ghost) * sn * 8, rbytes = size_t(ne) * sn * 8;
  {
    const char *u0 = reinterpret_cast<const char*>(U_dev), *r0 = reinterpret_cast<const char*>(R_dev);
    if (r0 < u0 + ubytes && u0 < r0 + rbytes) return fail(TDG_E_INVALID, "R_dev aliases U_dev");
  }
  std::lock_guard<std::mutex> lock(g_stage.call);
  if (int rc = ensure_staging()) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaStream_t cin = ctx->s_in[0], cout = ctx->s_out[0];
  // copy-in: piece i goes host -> staging[i % kStage] (pool) -> U_dev (DMA);
  // staging b is refilled once its previous DMA has finished
  cudaEventRecord(ctx->ev_s0, st);
  cudaStreamWaitEvent(cin, ctx->ev_s0, 0);
  cudaStreamWaitEvent(cout, ctx->ev_s0, 0);
  {
    int i = 0;
    for (size_t off = 0; off < ubytes; off += kStageBytes, ++i) {
      const size_t len = std::min(kStageBytes, ubytes - off);
      const int b = i % kStage;
      if (i >= kStage) cudaEventSynchronize(g_stage.ev[b]);
      par_copy(g_stage.buf[b], reinterpret_cast<const char*>(U_host) + off, len);
      cudaMemcpyAsync(reinterpret_cast<char*>(U_dev) + off, g_stage.buf[b], len,
                      cudaMemcpyHostToDevice, cin);
      cudaEventRecord(g_stage.ev[b], cin);
    }
  }
  cudaEventRecord(ctx->ev_s1, cin);
  cudaStreamWaitEvent(st, ctx->ev_s1, 0);
  // faces, then the volume kernel chunk by chunk (element-local: the same
  // bits as one launch)
  const int mode = mass_inverse ? 1 : 0;
  int rc = ctx->impl.run(ctx, U_dev, nullptr, R_dev, R_dev, 0.0, 0.0, 0.0, mode, 3, st);
  constexpr int NCH = tdg_ctx::kChunks;
  int64_t ck[NCH + 1];
  for (int k = 0; k <= NCH; ++k) ck[k] = chunk_start(ne, k);
  const bool faces = ctx->p.nif + ctx->p.nbf > 0;
  for (int k = 0; k < NCH && !rc; ++k) {
    rc = ctx->impl.volume(ctx, ck[k], ck[k + 1], U_dev, nullptr, R_dev, faces ? R_dev : nullptr,
                          0.0, 0.0, 0.0, mode, st);
    cudaEventRecord(ctx->ev_vol[k], st);
  }
  if (rc) {
    cudaStreamSynchronize(cin);
    return rc;
  }
  // copy-out pieces never straddle a volume chunk
  std::vector<Piece> pcs;
  for (int k = 0; k < NCH; ++k) {
    const size_t a = size_t(ck[k]) * sn * 8, b = size_t(ck[k + 1]) * sn * 8;
    for (size_t off = a; off < b; off += kStageBytes) pcs.push_back({off, std::min(kStageBytes, b - off), k});
  }
  auto issue = [&](size_t i) {
    const Piece& pc = pcs[i];
    const int b = int(i % kStage);
    cudaStreamWaitEvent(cout, ctx->ev_vol[pc.chunk], 0);
    cudaMemcpyAsync(g_stage.buf[b], reinterpret_cast<const char*>(R_dev) + pc.off, pc.len,
                    cudaMemcpyDeviceToHost, cout);
    cudaEventRecord(g_stage.ev[b], cout);
  };
  // the copy-in's staging DMAs are done before the first copy-out reuses them
  cudaStreamSynchronize(cin);
  for (size_t i = 0; i < pcs.size() && i < size_t(kStage); ++i) issue(i);
  for (size_t i = 0; i < pcs.size(); ++i) {
    const int b = int(i % kStage);
    cudaError_t e = cudaEventSynchronize(g_stage.ev[b]);
    if (e != cudaSuccess) return cuda_fail(e, "tdg_apply_host: copy-out");
    par_copy(reinterpret_cast<char*>(R_host) + pcs[i].off, g_stage.buf[b], pcs[i].len);
    if (i + kStage < pcs.size()) issue(i + kStage);
  }
  cudaEventRecord(ctx->ev_s1, cout);
  cudaStreamWaitEvent(st, ctx->ev_s1, 0);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "tdg_apply_host");
}
