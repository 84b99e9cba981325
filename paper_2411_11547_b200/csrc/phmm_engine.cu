// phmm_engine.cu — host engine + C-ABI of libphmm.so (see include/phmm.h).
//
// Host side (C++): validation, config binding (partition.py:20-37), pair enumeration
// (model.py:123-136), haplotype pairing + length binning + LPT ordering of work units,
// H2D upload, kernel launches on one stream, D2H and finishing (wavefront.py:428-434:
// flag acc<=0/non-finite, log10(acc) - s*log10 2 with glibc log10 like CPython math.log10).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/phmm.h"
#include "phmm_registry.h"

using namespace phmm;

namespace {

constexpr double kLog10_2 = 0.30102999566398120;   // np.log10(2.0), prob.py:41

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t n) {
    if (n <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr; cap = 0;
    size_t want = std::max<size_t>(n, 1);
    cudaError_t e = cudaMalloc(&p, want * sizeof(T));
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() { if (p) cudaFree(p); p = nullptr; cap = 0; }
};

// std::vector storage in pinned host memory: plan arrays are DMA'd without staging
template <class T>
struct PinnedAlloc {
  using value_type = T;
  PinnedAlloc() = default;
  template <class U> PinnedAlloc(const PinnedAlloc<U>&) {}
  // default-initialise (no zero fill of POD elements on resize)
  template <class U, class... A> void construct(U* p, A&&... a) {
    if constexpr (sizeof...(A) == 0) ::new ((void*)p) U;
    else ::new ((void*)p) U(std::forward<A>(a)...);
  }
  T* allocate(size_t n) {
    void* p = nullptr;
    if (cudaMallocHost(&p, n * sizeof(T)) != cudaSuccess) throw std::bad_alloc();
    return static_cast<T*>(p);
  }
  void deallocate(T* p, size_t) { cudaFreeHost(p); }
  template <class U> bool operator==(const PinnedAlloc<U>&) const { return true; }
  template <class U> bool operator!=(const PinnedAlloc<U>&) const { return false; }
};
template <class T> using PinnedVec = std::vector<T, PinnedAlloc<T>>;

// Stream tiling tables per mode (k_stream_<mode>.cu); kFast32's first kNumFastGeoms entries
// are the geometry table PHMM_FAST_GEOM ("PxK") selects from
constexpr int kNumFastGeoms = 13;
constexpr int kMaxTilings = 28;
static_assert(kNumStreamFast32 <= kMaxTilings, "tiling table");
const int kStreamTabN[4] = {kNumStreamFast32, kNumR64Geoms, kNumRX32Geoms, kNumR64Geoms};
const StreamKernel* stream_tab(int mode) {
  switch (mode) {
    case kFast32: return stream_table_fast32();
    case kFast64: return stream_table_fast64();
    case kExact32: return stream_table_exact32();
    default: return stream_table_exact64();
  }
}
const StreamKernel& striped_tab(int mode) {
  switch (mode) {
    case kFast32: return striped_fast32();
    case kFast64: return striped_fast64();
    case kExact32: return striped_exact32();
    default: return striped_exact64();
  }
}
// the tiling the striped instantiation of each mode corresponds to in its table
const int kStripedGeom[4] = {12, kNumR64Geoms - 1, kNumRX32Geoms - 1, kNumR64Geoms - 1};
// device counters: [0,4) ex32 counts, [4,8) ex64 counts, [8,12) ex32 work, [12,16) ex64
// work, 16 inline guard-band pairs, [20,24) fx64 counts, [24,28) fx64 work, then the
// device-built stream lists (counts[8], hap count, overflow) and their work counters, then
// one work counter per planned stream bin
constexpr int kCtrR64 = 32, kCtrRX32 = 44, kCtrR64Work = 56, kCtrRX32Work = 64;
constexpr int kCtrR64b = 72, kCtrR64bWork = 80;   // second-stage striped FP64 units: counts, work
constexpr int kBinCounters = 96;                  // fixed counter slots before the per-bin counters
constexpr int64_t kBigCallPairs = 1 << 20;        // phmm_score pipelines calls above this
constexpr int64_t kMidCallPairs = 1 << 16;        // device-built retry units grow above this
constexpr int kFinishThreads = 16;                // host threads finishing log10 in phmm_fetch
// scratch bound for boundary columns of long haplotypes (striped stream bins, post-pass);
// contexts of a budgeted phmm_score use an eighth of their chunk budget instead
constexpr size_t kColBudget = (size_t)1 << 30;
// device bytes per pair a prepare can allocate (acc, status, stream entry, the device-built
// retry units / entries and per-pair lists, each sized for every pair), for chunk budgets
constexpr int64_t kDevBytesPerPair = 200;

int stream_cap(int P) { return stream_cap_of(P); }

// PHMM_OCC_CAP=n (experiments): at most n CTAs per SM for every stream-kernel grid
int occ_cap(int occ) {
  static int v = -1;
  if (v < 0) {
    const char* env = getenv("PHMM_OCC_CAP");
    v = env ? std::max(1, atoi(env)) : 1 << 20;
  }
  return std::min(occ, v);
}

int exact_slot_host(int m) { return (m + 1 <= 32) ? 0 : (m + 1 <= 64) ? 1 : (m + 1 <= 128) ? 2 : 3; }

int forced_geom() {
  static int g = -2;
  if (g == -2) {
    g = -1;
    const char* env = getenv("PHMM_FAST_GEOM");      // tuning knob: "PxK"
    int P = 0, K = 0;
    if (env && sscanf(env, "%dx%d", &P, &K) == 2)
      for (int i = 0; i < kNumFastGeoms; ++i)
        if (stream_table_fast32()[i].P == P && stream_table_fast32()[i].K == K) g = i;
  }
  return g;
}

// Cost of streaming a read's haplotypes (lengths summing to `total`, longest `nmax`) on
// tiling g: units of two lanes of ~total/2 rows, split when a lane would exceed the
// tiling's row-code capacity or `lane_rows`, the call's lane-length budget (small calls
// split units further, below).  INT64_MAX: excluded by PHMM_FAST_GEOM.
int64_t stream_geom_cost(int mode, int g, int64_t total, int nmax, int64_t lane_rows = INT64_MAX) {
  constexpr int64_t kInf = INT64_MAX;
  const int fg = forced_geom();
  if (mode == kFast32 && fg >= 0 && g != fg) return kInf;
  const int64_t P = stream_tab(mode)[g].P, K = stream_tab(mode)[g].K;
  // a haplotype longer than the row capacity streams alone in its lane (ring mode)
  const int64_t cap = std::max<int64_t>(nmax, std::min<int64_t>(stream_cap((int)P), std::max<int64_t>(nmax, lane_rows)));
  const int64_t units = (total + 2 * cap - 1) / (2 * cap);
  const int64_t rows = std::min<int64_t>(cap, (total + 2 * units - 1) / (2 * units));
  const int64_t c = units * P * (2 * K + 5) * (rows + P - 1);     // 2 x (K + 2.5) per thread-row
  // 4-thread sub-warps run at ~70 % of the per-cell rate the model gives them (8 units per
  // warp: the warp steps through the union of their event windows); x1.3 hands reads of
  // 48-63 bases to (8,8) instead of (4,16): c5 FP32 phase 132.2 -> 131.4 ms
  return (mode == kFast32 && P == 4) ? c * 13 / 10 : c;
}
int choose_stream_geom(int mode, int m, int64_t total, int nmax, int64_t lane_rows) {
  int64_t best = INT64_MAX;
  int bi = -1;
  for (int g = 0; g < kStreamTabN[mode]; ++g) {
    if (m + 1 > stream_tab(mode)[g].P * stream_tab(mode)[g].K) continue;
    const int64_t cost = stream_geom_cost(mode, g, total, nmax, lane_rows);
    if (cost < best) { best = cost; bi = g; }
  }
  return bi;
}
constexpr int kStripedBin = 1 << 10;          // geometry code of a striped bin
const StreamKernel& skern(int mode, int geom) {
  return (geom & kStripedBin) ? striped_tab(mode) : stream_tab(mode)[geom];
}
// column rows a striped unit of tiling P with lanes of <= max_rows rows can need (the
// row-0 slot + one spare)
int col_rows_for(int P, int max_rows) { return std::max(stream_cap_of(P), max_rows) + 2; }
constexpr int kR64MaxW = 256, kRX32MaxW = 512;   // widest FP64 / exact-FP32 retry tilings

constexpr int kMaxScoreChunks = 8;
// Small persistent worker pool for host-side data-parallel loops (result finishing).
class WorkerPool {
 public:
  explicit WorkerPool(int n) {
    for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~WorkerPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  int size() const { return (int)workers_.size(); }
  // runs fn(i) for i in [0, tasks) on the workers and the caller; returns when all are done
  void run(int tasks, const std::function<void(int)>& fn) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      tasks_ = tasks;
      next_ = 0;
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return done_ == tasks_; });
    fn_ = nullptr;
  }

 private:
  void work() {
    for (;;) {
      int i;
      const std::function<void(int)>* f;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (!fn_ || next_ >= tasks_) return;
        i = next_++;
        f = fn_;
      }
      (*f)(i);
      std::lock_guard<std::mutex> lk(mu_);
      if (++done_ == tasks_) done_cv_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int tasks_ = 0, next_ = 0, done_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// PHMM_TRACE=1: wall-clock breakdown of the host phases on stderr
struct Trace {
  bool on;
  std::chrono::steady_clock::time_point last;
  std::string buf;
  Trace() : on(getenv("PHMM_TRACE") != nullptr), last(std::chrono::steady_clock::now()) {}
  void mark(const char* what) {
    if (!on) return;
    auto now = std::chrono::steady_clock::now();
    char tmp[64];
    snprintf(tmp, sizeof(tmp), " %s=%.3f", what, std::chrono::duration<double, std::milli>(now - last).count());
    buf += tmp;
    last = now;
  }
  void print(const char* phase) {
    if (on) fprintf(stderr, "[phmm %s]%s ms\n", phase, buf.c_str());
  }
};

}  // namespace

struct phmm_ctx {
  int device = 0;
  int num_sms = 148;
  size_t total_mem = 0;                      // device memory (bytes)
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_start = nullptr, ev_fast0 = nullptr, ev_fast1 = nullptr, ev_end = nullptr;   // execute
  cudaEvent_t ev_post1 = nullptr;                       // execute: end of the concurrent post-pass
  cudaEvent_t ev_span0 = nullptr;                       // phmm_score chunked: first chunk's execute start
  cudaEvent_t ev_up0 = nullptr, ev_up1 = nullptr;       // prepare: uploads + device validation
  cudaEvent_t ev_d0 = nullptr, ev_d1 = nullptr;         // fetch: D2H of the results
  cudaEvent_t ev_pre = nullptr;
  static constexpr int kAux = 16;             // side streams: kernels of a phase run concurrently
  cudaStream_t aux[kAux] = {};
  cudaEvent_t ev_join[kAux] = {};
  cudaEvent_t ev_x32[kAux] = {};              // execute: exact-FP32 post-pass launches done
  cudaStream_t r64b_st[kNumR64Geoms] = {};    // second-stage FP64 units, one stream per tiling
  cudaEvent_t ev_r64b[kNumR64Geoms] = {};
  std::string err;
  std::vector<double> lut;

  // device buffers
  DBuf<int8_t> d_rbases, d_hbases;
  DBuf<uint8_t> d_bq, d_iq, d_dq, d_gq, d_status, d_rflags;
  DBuf<int64_t> d_roff, d_hoff;
  DBuf<int> d_read_m, d_read_scale, d_read_ncap, d_counters, d_vflag;
  DBuf<float> d_gsum;
  DBuf<double> d_lut, d_acc;
  DBuf<StreamUnit> d_sunits;
  DBuf<StreamHap> d_shaps;
  DBuf<StreamUnit> d_r64u[kNumR64Geoms], d_rx32u[kNumRX32Geoms];
  DBuf<StreamHap> d_r64h, d_rx32h;
  DBuf<ExactItem> d_ex32[kNumExactP], d_ex64[kNumExactP], d_fx64[kNumExactP];
  DBuf<double> d_cold;
  std::unique_ptr<WorkerPool> pool;         // host finishing threads (lazy)
  int* h_counts = nullptr;   // pinned: initial list counts (8) + zeros for work counters
  int* h_vflag = nullptr;    // pinned: device validation flag
  bool async = false;        // chunk contexts of phmm_score: no host syncs in prepare/execute
  phmm_ctx* parent = nullptr;
  int budget_div = 1;        // chunk contexts: number of chunks sharing the band budget
  int64_t device_budget = 0; // phmm_set_device_budget: bound on the device working set of phmm_score (0: none)
  int pipeline = 0;          // phmm_set_pipeline: 0 automatic, 1 never, n equal chunks
  size_t col_budget = kColBudget;        // boundary-column scratch bound of this context
  std::vector<phmm_ctx*> chunks;             // chunk contexts (phmm_score pipelining), lazy
  PinnedVec<int64_t> c_roff, c_hoff;         // chunk views: rebased offsets (pinned: async H2D)
  std::vector<int64_t> c_bro, c_bho;
  double* h_acc = nullptr;   // pinned result staging (phmm_fetch)
  uint8_t* h_st = nullptr;
  int64_t h_res_cap = 0;

  // plan (host)
  bool prepared = false, executed = false;
  int64_t num_pairs = 0;
  int64_t num_reads = 0, num_haps = 0, num_batches = 0;
  std::vector<int64_t> batch_read_off, batch_hap_off, hap_len;
  std::vector<int> read_m, read_scale, read_cfg;   // read_cfg -1 = too small
  unsigned r64_geoms = 0, rx32_geoms = 0;   // device-built unit tilings that can get work
  struct SBin {
    int mode;
    int geom;
    int64_t count = 0;                      // units of this tiling
    int64_t dev_off = 0;                    // first unit in h_sunits / d_sunits
    int64_t col_off = -1;                   // striped units: column buffer (bytes), else -1
    int grid = 0;
    int max_rows = 0;                       // longest lane of the bin's units
  };
  std::vector<SBin> sbins;
  DBuf<unsigned char> d_colstream;          // boundary columns of striped stream units
  int64_t r64_col_off[8] = {-1, -1, -1, -1, -1, -1, -1, -1}, rx32_col_off[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
  std::vector<int> sbin_order;
  std::vector<StreamUnit> su_all;           // planning scratch (persistent capacity)
  std::vector<uint8_t> su_bin;
  std::vector<int> su_cnt;
  PinnedVec<StreamHap> shaps;               // persistent capacity (pinned)
  PinnedVec<StreamUnit> h_sunits;           // LPT-ordered stream units, all bins
  PinnedVec<int> h_rmeta;                   // read m | scale | ncap
  int max_n = 1;
  int flags = 0;
  int list_cap[kNumExactP] = {0, 0, 0, 0};
  int64_t h2d_bytes = 0;
  int64_t hap_bytes = 0, read_bytes = 0;
  double plan_ms = 0.0, h2d_ms = 0.0;
  int last_launches = 0;
  int post_grid = 0;                         // CTAs of the per-pair post-pass kernels
  int r64_grid = 0, rx32_grid = 0;           // CTAs of the striped retry launches
  float last_dev_ms = 0.f, last_fast_ms = 0.f;
  float last_phase_ms[4] = {0.f, 0.f, 0.f, 0.f};   // precompute, FP32 stream, post-pass (a), (b)+(c)
  EngineDev dev{};

  int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    err = buf;
    return code;
  }
  int cuda_fail(cudaError_t e, const char* what) {
    return fail(PHMM_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  }
};

#define CK(call)                                                        \
  do {                                                                  \
    cudaError_t _e = (call);                                            \
    if (_e != cudaSuccess) return ctx->cuda_fail(_e, #call);            \
  } while (0)

extern "C" {

int phmm_abi_version(void) { return PHMM_ABI_VERSION; }

static int init_ctx(phmm_ctx* ctx, int device);

int phmm_create(phmm_ctx** out, int device, const double* phred_lut) {
  if (!out || !phred_lut) return PHMM_ERR_INVALID;
  *out = nullptr;
  phmm_ctx* ctx = new (std::nothrow) phmm_ctx();
  if (!ctx) return PHMM_ERR_NOMEM;
  ctx->device = device;
  ctx->lut.assign(phred_lut, phred_lut + 94);
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || device < 0 || device >= ndev) {
    *out = ctx;
    ctx->fail(PHMM_ERR_CUDA, "no CUDA device %d (%s)", device,
              e != cudaSuccess ? cudaGetErrorString(e) : "out of range");
    return PHMM_ERR_CUDA;
  }
  *out = ctx;
  return init_ctx(ctx, device);
}

static int init_ctx(phmm_ctx* ctx, int device) {
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return ctx->fail(PHMM_ERR_CUDA, "device %s is sm_%d%d; libphmm is built for sm_100a",
                                         prop.name, prop.major, prop.minor);
  ctx->num_sms = prop.multiProcessorCount;
  ctx->total_mem = prop.totalGlobalMem;
  CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ctx->ev_pre, cudaEventDisableTiming));
  for (int a = 0; a < phmm_ctx::kAux; ++a) {
    CK(cudaStreamCreateWithFlags(&ctx->aux[a], cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_join[a], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_x32[a], cudaEventDisableTiming));
  }
  for (int g = 0; g < kNumR64Geoms; ++g) {
    CK(cudaStreamCreateWithFlags(&ctx->r64b_st[g], cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_r64b[g], cudaEventDisableTiming));
  }
  CK(cudaEventCreate(&ctx->ev_start));
  CK(cudaEventCreate(&ctx->ev_fast0));
  CK(cudaEventCreate(&ctx->ev_fast1));
  CK(cudaEventCreate(&ctx->ev_end));
  CK(cudaEventCreate(&ctx->ev_post1));
  CK(cudaEventCreate(&ctx->ev_span0));
  CK(cudaEventCreate(&ctx->ev_up0));
  CK(cudaEventCreate(&ctx->ev_up1));
  CK(cudaEventCreate(&ctx->ev_d0));
  CK(cudaEventCreate(&ctx->ev_d1));
  CK(cudaMallocHost(&ctx->h_counts, kBinCounters * sizeof(int)));
  CK(cudaMallocHost(&ctx->h_vflag, sizeof(int)));
  CK(ctx->d_lut.ensure(94));
  CK(cudaMemcpy(ctx->d_lut.p, ctx->lut.data(), 94 * sizeof(double), cudaMemcpyHostToDevice));
  for (int md = 0; md < 4; ++md) {
    for (int g = 0; g < kStreamTabN[md]; ++g) {
      const StreamKernel& k = stream_tab(md)[g];
      CK(cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.smem));
      // one shared-memory carveout for every stream kernel: CTAs of different tilings can
      // share an SM without an L1/shared reconfiguration
      if (!getenv("PHMM_NO_CARVEOUT"))
        CK(cudaFuncSetAttribute(k.fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    }
    CK(cudaFuncSetAttribute(striped_tab(md).fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)striped_tab(md).smem));
  }
  CK(aux_set_attributes());
  return PHMM_SUCCESS;
}

int phmm_destroy(phmm_ctx* ctx) {
  if (!ctx) return PHMM_SUCCESS;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  ctx->d_rbases.release(); ctx->d_hbases.release(); ctx->d_bq.release(); ctx->d_iq.release();
  ctx->d_dq.release(); ctx->d_gq.release(); ctx->d_status.release(); ctx->d_rflags.release();
  ctx->d_roff.release(); ctx->d_hoff.release(); ctx->d_read_m.release(); ctx->d_read_scale.release();
  ctx->d_read_ncap.release(); ctx->d_counters.release(); ctx->d_vflag.release();
  ctx->d_colstream.release(); ctx->d_gsum.release(); ctx->d_lut.release();
  ctx->d_acc.release(); ctx->d_sunits.release(); ctx->d_shaps.release();
  for (int g = 0; g < kNumR64Geoms; ++g) ctx->d_r64u[g].release();
  for (int g = 0; g < kNumRX32Geoms; ++g) ctx->d_rx32u[g].release();
  ctx->d_r64h.release();
  ctx->d_rx32h.release(); ctx->d_cold.release();
  for (int s = 0; s < kNumExactP; ++s) { ctx->d_ex32[s].release(); ctx->d_ex64[s].release(); ctx->d_fx64[s].release(); }
  for (phmm_ctx* c : ctx->chunks) phmm_destroy(c);
  ctx->chunks.clear();
  if (ctx->h_counts) cudaFreeHost(ctx->h_counts);
  if (ctx->h_vflag) cudaFreeHost(ctx->h_vflag);
  if (ctx->h_acc) cudaFreeHost(ctx->h_acc);
  if (ctx->h_st) cudaFreeHost(ctx->h_st);
  ctx->h_counts = nullptr;
  if (ctx->ev_start) cudaEventDestroy(ctx->ev_start);
  if (ctx->ev_fast0) cudaEventDestroy(ctx->ev_fast0);
  if (ctx->ev_fast1) cudaEventDestroy(ctx->ev_fast1);
  if (ctx->ev_end) cudaEventDestroy(ctx->ev_end);
  for (cudaEvent_t e : {ctx->ev_up0, ctx->ev_up1, ctx->ev_d0, ctx->ev_d1, ctx->ev_post1, ctx->ev_span0})
    if (e) cudaEventDestroy(e);
  if (ctx->ev_pre) cudaEventDestroy(ctx->ev_pre);
  for (int a = 0; a < phmm_ctx::kAux; ++a) {
    if (ctx->aux[a]) { cudaStreamSynchronize(ctx->aux[a]); cudaStreamDestroy(ctx->aux[a]); }
    if (ctx->ev_join[a]) cudaEventDestroy(ctx->ev_join[a]);
    if (ctx->ev_x32[a]) cudaEventDestroy(ctx->ev_x32[a]);
  }
  for (int g = 0; g < kNumR64Geoms; ++g) {
    if (ctx->r64b_st[g]) { cudaStreamSynchronize(ctx->r64b_st[g]); cudaStreamDestroy(ctx->r64b_st[g]); }
    if (ctx->ev_r64b[g]) cudaEventDestroy(ctx->ev_r64b[g]);
  }
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return PHMM_SUCCESS;
}

const char* phmm_last_error(const phmm_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

static int prepare_impl(phmm_ctx* ctx, const phmm_input* in, const phmm_options* opt, int64_t* num_pairs_out);

// waits for the prepare's uploads and the device content checks (k_validate)
static int check_validation(phmm_ctx* ctx) {
  CK(cudaEventSynchronize(ctx->ev_up1));
  const int vbad = *ctx->h_vflag;
  if (vbad & 1) return ctx->fail(PHMM_ERR_INVALID, "base code outside A,C,G,T,N (0..4)");
  if (vbad & 2) return ctx->fail(PHMM_ERR_INVALID, "quality values must be in [0, 93]");
  return PHMM_SUCCESS;
}

int phmm_prepare(phmm_ctx* ctx, const phmm_input* in, const phmm_options* opt, int64_t* num_pairs_out) {
  if (!ctx) return PHMM_ERR_INVALID;
  try {
    return prepare_impl(ctx, in, opt, num_pairs_out);
  } catch (const std::bad_alloc&) {
    return ctx->fail(PHMM_ERR_NOMEM, "host allocation failed");
  }
}

static int prepare_impl(phmm_ctx* ctx, const phmm_input* in, const phmm_options* opt, int64_t* num_pairs_out) {
  if (!in || !opt) return ctx->fail(PHMM_ERR_INVALID, "null input/options");
  auto t0 = std::chrono::steady_clock::now();
  Trace trace;
  CK(cudaSetDevice(ctx->device));
  ctx->prepared = false;
  ctx->executed = false;
  const int64_t R = in->num_reads, H = in->num_haps, B = in->num_batches;
  if (R < 0 || H < 0 || B < 0) return ctx->fail(PHMM_ERR_INVALID, "negative counts");
  if (opt->num_configs < 0 || (opt->num_configs > 0 && (!opt->p || !opt->k || !opt->precision || !opt->scale_log2)))
    return ctx->fail(PHMM_ERR_INVALID, "bad config table");
  // ---- structure validation
  if (B > 0 && (!in->batch_read_off || !in->batch_hap_off)) return ctx->fail(PHMM_ERR_INVALID, "null batch offsets");
  if (B > 0) {
    if (in->batch_read_off[0] != 0 || in->batch_hap_off[0] != 0 || in->batch_read_off[B] != R ||
        in->batch_hap_off[B] != H)
      return ctx->fail(PHMM_ERR_INVALID, "batch offsets do not cover the read/hap arrays");
    for (int64_t b = 0; b < B; ++b)
      if (in->batch_read_off[b + 1] <= in->batch_read_off[b] || in->batch_hap_off[b + 1] <= in->batch_hap_off[b])
        return ctx->fail(PHMM_ERR_INVALID, "batch %lld must contain at least one read and one haplotype",
                         (long long)b);
  } else if (R != 0 || H != 0) {
    return ctx->fail(PHMM_ERR_INVALID, "reads/haps given without batches");
  }
  const int64_t* roff = in->read_off;
  const int64_t* hoff = in->hap_off;
  if (R > 0 && (!roff || roff[0] != 0)) return ctx->fail(PHMM_ERR_INVALID, "read offsets must start at 0");
  if (H > 0 && (!hoff || hoff[0] != 0)) return ctx->fail(PHMM_ERR_INVALID, "hap offsets must start at 0");
  for (int64_t r = 0; r < R; ++r)
    if (roff[r + 1] <= roff[r]) return ctx->fail(PHMM_ERR_INVALID, "read %lld must contain at least one base", (long long)r);
  for (int64_t h = 0; h < H; ++h)
    if (hoff[h + 1] <= hoff[h]) return ctx->fail(PHMM_ERR_INVALID, "haplotype %lld must contain at least one base", (long long)h);
  const int64_t RL = R ? roff[R] : 0, HL = H ? hoff[H] : 0;
  if (RL > 0 && (!in->read_bases || !in->base_qual || !in->ins_qual || !in->del_qual || !in->gcp_qual))
    return ctx->fail(PHMM_ERR_INVALID, "null read arrays");
  if (HL > 0 && !in->hap_bases) return ctx->fail(PHMM_ERR_INVALID, "null haplotype bases");
  for (int c = 0; c < opt->num_configs; ++c) {
    if (opt->p[c] < 1 || opt->k[c] < 1 || (opt->precision[c] != 0 && opt->precision[c] != 1) || opt->scale_log2[c] < 0)
      return ctx->fail(PHMM_ERR_INVALID, "invalid config %d", c);
  }
  ctx->flags = opt->flags;
  ctx->hap_bytes = HL;
  ctx->read_bytes = RL;
  ctx->num_reads = R; ctx->num_haps = H; ctx->num_batches = B;
  ctx->batch_read_off.assign(in->batch_read_off, in->batch_read_off + (B ? B + 1 : 0));
  ctx->batch_hap_off.assign(in->batch_hap_off, in->batch_hap_off + (B ? B + 1 : 0));
  ctx->hap_len.resize(H);
  for (int64_t h = 0; h < H; ++h) ctx->hap_len[h] = hoff[h + 1] - hoff[h];

  trace.mark("validate");
  // ---- raw inputs go to the device first (async): the copy overlaps the host planning
  // below; their content checks run on the device (k_validate) at the end of prepare
  int64_t bytes = 0;
  auto up = [&](auto& buf, const auto* src, size_t n) -> cudaError_t {
    cudaError_t e = buf.ensure(n);
    if (e != cudaSuccess || n == 0) return e;
    bytes += (int64_t)(n * sizeof(*src));
    return cudaMemcpyAsync(buf.p, src, n * sizeof(*src), cudaMemcpyHostToDevice, ctx->stream);
  };
  CK(cudaEventRecord(ctx->ev_up0, ctx->stream));
  CK(up(ctx->d_rbases, in->read_bases, RL));
  CK(up(ctx->d_bq, in->base_qual, RL));
  CK(up(ctx->d_iq, in->ins_qual, RL));
  CK(up(ctx->d_dq, in->del_qual, RL));
  CK(up(ctx->d_gq, in->gcp_qual, RL));
  trace.mark("h2d-reads");
  CK(up(ctx->d_roff, roff, R ? R + 1 : 0));
  CK(ctx->d_hbases.ensure((size_t)HL + 16));     // + 16: the stream kernels read 16-byte chunks
  CK(up(ctx->d_hbases, in->hap_bases, HL));
  CK(up(ctx->d_hoff, hoff, H ? H + 1 : 0));

  trace.mark("h2d-issue");
  // ---- config binding: smallest p*k >= m, ties to fewer lanes (partition.py:20-37)
  std::vector<int> order(opt->num_configs);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    const int64_t ma = (int64_t)opt->p[a] * opt->k[a], mb = (int64_t)opt->p[b] * opt->k[b];
    return ma != mb ? ma < mb : opt->p[a] < opt->p[b];
  });
  ctx->read_m.resize(R); ctx->read_scale.resize(R); ctx->read_cfg.resize(R);
  std::vector<int> read_ncap(R, 1);
  // host worker pool (shared with the chunk contexts of a pipelined call): large calls bind
  // and plan on it
  WorkerPool* pool = nullptr;
  if (R >= (1 << 13)) {
    phmm_ctx* owner = ctx->parent ? ctx->parent : ctx;
    if (!owner->pool) {
      const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
      owner->pool.reset(new WorkerPool(std::min(hw, kFinishThreads) - 1));
    }
    pool = owner->pool.get();
  }
  auto par_for = [&](int64_t n, int tasks, const std::function<void(int64_t, int64_t)>& body) {
    if (!pool || tasks <= 1 || n < 2 * tasks) { body(0, n); return; }
    std::function<void(int)> task = [&](int i) { body(n * i / tasks, n * (i + 1) / tasks); };
    pool->run(tasks, task);
  };
  std::vector<int> too_long;
  std::mutex too_long_mu;
  par_for(R, pool ? pool->size() + 1 : 1, [&](int64_t a, int64_t z) {
    int64_t memo_m = -1;
    int memo_cfg = -1;
    for (int64_t r = a; r < z; ++r) {
      const int64_t m = roff[r + 1] - roff[r];
      if (m > (int64_t)1 << 30) {
        std::lock_guard<std::mutex> lk(too_long_mu);
        too_long.push_back((int)r);
        continue;
      }
      ctx->read_m[r] = (int)m;
      if (m != memo_m) {                               // reads of a batch often share m
        memo_cfg = -1;
        for (int c : order)
          if ((int64_t)opt->p[c] * opt->k[c] >= m) { memo_cfg = c; break; }
        memo_m = m;
      }
      ctx->read_cfg[r] = memo_cfg;
      ctx->read_scale[r] = memo_cfg >= 0 ? opt->scale_log2[memo_cfg] : 0;
    }
  });
  if (!too_long.empty()) return ctx->fail(PHMM_ERR_INVALID, "read too long");
  trace.mark("bind");
  // ---- pairs, hap pairing, units
  int64_t N = 0;
  for (int64_t b = 0; b < B; ++b)
    N += (ctx->batch_read_off[b + 1] - ctx->batch_read_off[b]) * (ctx->batch_hap_off[b + 1] - ctx->batch_hap_off[b]);
  if (N > INT32_MAX - 1) return ctx->fail(PHMM_ERR_INVALID, "too many pairs in one call (%lld)", (long long)N);
  ctx->num_pairs = N;
  const bool exact_mode = (opt->flags & PHMM_FLAG_EXACT) != 0;
  // stream units address reads/haplotypes with 32-bit offsets (phmm_score chunks larger calls)
  if (RL >= INT32_MAX || HL >= INT32_MAX)
    return ctx->fail(PHMM_ERR_INVALID, "one prepare holds < 2 GiB of read / haplotype bases; use phmm_score "
                                       "(which streams larger inputs in chunks)");
  ctx->sbins.clear();
  ctx->r64_geoms = ctx->rx32_geoms = 0;
  ctx->su_all.clear();
  ctx->su_bin.clear();
  ctx->shaps.clear();
  int sbin_index[4 * kMaxTilings];
  std::fill(sbin_index, sbin_index + 4 * kMaxTilings, -1);
  int64_t slot_pairs[kNumExactP] = {0, 0, 0, 0};
  int64_t r64_pairs[8] = {0}, rx32_pairs[8] = {0};
  bool long64 = false, long32 = false;          // streamed reads that stripe in the retry kernels
  int64_t stripe_pairs = 0;                     // pairs of reads that stripe in the per-pair post-pass
  int max_n = 1;
  struct LaneTemplate {
    std::vector<int> lanes[2];
    int rows[2] = {0, 0};
  };
  // per mode: tiling tables sorted by width (the choice depends on m only through
  // W >= m + 1), best tiling per width and lane templates, both cached per batch
  struct ModePlan {
    int n = 0;
    int wsort[kMaxTilings], wsorted[kMaxTilings], best_from[kMaxTilings];
    bool tvalid[kMaxTilings];
    std::vector<LaneTemplate> tmpls[kMaxTilings];
    int tmpl_m = -1, tmpl_geom = -2;
  };
  ModePlan mp0[4];                              // tiling tables (copied per planning part)
  for (int md = 0; md < 4; ++md) {
    ModePlan& M = mp0[md];
    M.n = kStreamTabN[md];
    for (int g = 0; g < M.n; ++g) M.wsort[g] = g;
    std::sort(M.wsort, M.wsort + M.n, [&](int x, int y) {
      return stream_tab(md)[x].P * stream_tab(md)[x].K < stream_tab(md)[y].P * stream_tab(md)[y].K;
    });
    for (int i = 0; i < M.n; ++i) M.wsorted[i] = stream_tab(md)[M.wsort[i]].P * stream_tab(md)[M.wsort[i]].K;
  }
  // Lane budget: a call too small to fill the GPU with long lanes (few pairs, long
  // haplotypes: c4, c3) splits its units until there are ~6 per sub-warp slot (#SM x 8
  // warps x 2 sub-warps; PHMM_LANE_UNITS): the last wave's tail, not per-unit overhead,
  // bounds such calls (c3: 2 -> 6 per slot, FP32 phase -6 %; c2 unchanged, 8 is worse).
  // Large calls keep the row capacity as the only limit.  Per batch: first pair id and
  // first stream entry.
  int64_t lane_rows = INT64_MAX;
  std::vector<int64_t> bgid(B + 1, 0), bsh(B + 1, 0);
  {
    int64_t all_rows = 0;
    for (int64_t b = 0; b < B; ++b) {
      const int64_t r0 = ctx->batch_read_off[b], r1 = ctx->batch_read_off[b + 1];
      int64_t hs = 0, live = 0;
      for (int64_t h = ctx->batch_hap_off[b]; h < ctx->batch_hap_off[b + 1]; ++h) hs += ctx->hap_len[h];
      for (int64_t r = r0; r < r1; ++r) live += ctx->read_cfg[r] >= 0;
      const int64_t nh = ctx->batch_hap_off[b + 1] - ctx->batch_hap_off[b];
      all_rows += hs * (r1 - r0);
      bgid[b + 1] = bgid[b] + nh * (r1 - r0);
      bsh[b + 1] = bsh[b] + nh * live;
    }
    static const int lane_units = [] {          // units per sub-warp slot targeted (PHMM_LANE_UNITS)
      const char* e = getenv("PHMM_LANE_UNITS");
      return e ? std::max(1, atoi(e)) : 6;
    }();
    if (!getenv("PHMM_NO_LANE_BUDGET")) lane_rows = all_rows / (2 * lane_units * (int64_t)ctx->num_sms * 16);
  }
  ctx->shaps.resize(bsh[B]);                     // default-initialised (PinnedAlloc::construct)
  // Units of batches [b0, b1) into one part; parts are planned concurrently on the worker
  // pool and merged in batch order, so the plan equals a sequential pass over the batches.
  struct PlanPart {
    std::vector<StreamUnit> su;
    std::vector<uint16_t> key;                   // per unit: mode * kMaxTilings + template slot
    std::vector<int> keys;                       // keys in order of first appearance
    int key_geom[4 * kMaxTilings];
    int key_rows[4 * kMaxTilings];
    int64_t slot_pairs[kNumExactP] = {0, 0, 0, 0};
    int64_t r64_pairs[8] = {0}, rx32_pairs[8] = {0};
    bool long64 = false, long32 = false;         // streamed reads that stripe in the retry kernels
    int64_t stripe_pairs = 0;
    unsigned r64_geoms = 0, rx32_geoms = 0;
    int max_n = 1;
  };
  auto plan_range = [&](int64_t b0, int64_t b1, PlanPart& pp) {
    std::fill(pp.key_geom, pp.key_geom + 4 * kMaxTilings, -1);
    std::fill(pp.key_rows, pp.key_rows + 4 * kMaxTilings, 0);
    std::vector<int> hidx;
    ModePlan mp[4];
    for (int md = 0; md < 4; ++md) mp[md] = mp0[md];
    StreamHap* sh_out = ctx->shaps.data() + bsh[b0];
    int64_t gid = bgid[b0];
    for (int64_t b = b0; b < b1; ++b) {
      const int64_t r0 = ctx->batch_read_off[b], r1 = ctx->batch_read_off[b + 1];
      const int64_t h0 = ctx->batch_hap_off[b], h1 = ctx->batch_hap_off[b + 1];
      const int64_t nh = h1 - h0;
      int ncap = 1;
      int64_t batch_total = 0;
      for (int64_t h = h0; h < h1; ++h) {
        ncap = (int)std::max<int64_t>(ncap, ctx->hap_len[h]);
        batch_total += ctx->hap_len[h];
      }
      pp.max_n = std::max(pp.max_n, ncap);
      for (int md = 0; md < 4; ++md) {
        mp[md].tmpl_m = -1;
        mp[md].tmpl_geom = -2;
        std::fill(mp[md].tvalid, mp[md].tvalid + kMaxTilings, false);
        std::fill(mp[md].best_from, mp[md].best_from + kMaxTilings, -2);
      }
      hidx.resize(nh);
      std::iota(hidx.begin(), hidx.end(), (int)h0);
      std::stable_sort(hidx.begin(), hidx.end(), [&](int a, int c) { return ctx->hap_len[a] > ctx->hap_len[c]; });
      for (int64_t r = r0; r < r1; ++r, gid += nh) {
        read_ncap[r] = ncap;
        const int cfg = ctx->read_cfg[r];
        if (cfg < 0) continue;                         // config-too-small: host-side status
        const int m = ctx->read_m[r];
        const int scale = opt->scale_log2[cfg];
        const bool f64 = opt->precision[cfg] == 1;
        const bool exact = f64 || exact_mode || scale > 126;
        const int mode = f64 ? kExact64 : exact ? kExact32 : kFast32;
        pp.slot_pairs[exact_slot_host(m)] += nh;      // any pair may land in its slot's lists
        if (m + 1 > 32 * kExactK) pp.stripe_pairs += nh;
        ModePlan& M = mp[mode];
        if (m != M.tmpl_m) {                           // lane template per (batch, tiling)
          M.tmpl_m = m;
          int sg = -1;
          for (int i = 0; i < M.n; ++i)                // best tiling of the narrowest width >= m+1
            if (M.wsorted[i] >= m + 1) {
              if (M.best_from[i] == -2) M.best_from[i] = choose_stream_geom(mode, M.wsorted[i] - 1, batch_total, ncap, lane_rows);
              sg = M.best_from[i];
              break;
            }
          if (sg < 0) sg = kStripedBin | kStripedGeom[mode];   // longer than every tiling: stripes
          M.tmpl_geom = sg;
          const int ts = (sg & kStripedBin) ? kMaxTilings - 1 : sg;   // template cache slot
          if (!M.tvalid[ts]) {
            M.tvalid[ts] = true;
            std::vector<LaneTemplate>& tmpl = M.tmpls[ts];
            tmpl.clear();
            // greedy LPT over the length-sorted haplotypes: each to the lighter lane; a
            // new unit when a lane would exceed the tiling's row capacity or the call's
            // lane budget
            const int cap = (int)std::min<int64_t>(stream_cap(skern(mode, sg).P), std::max<int64_t>(lane_rows, 1));
            // kFast32 lanes separate their haplotypes by one idle row (SepRows, phmm_kernels.cuh)
            const int sep = mode == kFast32 ? 1 : 0;
            tmpl.emplace_back();
            for (int64_t x = 0; x < nh; ++x) {
              const int h = hidx[x];
              const int n = (int)ctx->hap_len[h];
              LaneTemplate* t = &tmpl.back();
              int ln = t->rows[0] <= t->rows[1] ? 0 : 1;
              if ((t->rows[ln] > 0 && t->rows[ln] + sep + n > cap) || (int)t->lanes[ln].size() >= kStreamMaxLaneHaps) {
                tmpl.emplace_back();
                t = &tmpl.back();
                ln = 0;
              }
              t->rows[ln] += n + (t->rows[ln] > 0 ? sep : 0);
              t->lanes[ln].push_back(h);
            }
          }
        }
        const int ts = (M.tmpl_geom & kStripedBin) ? kMaxTilings - 1 : M.tmpl_geom;
        const std::vector<LaneTemplate>& tmpl = M.tmpls[ts];
        const int key = mode * kMaxTilings + ts;
        if (pp.key_geom[key] < 0) {
          pp.key_geom[key] = M.tmpl_geom;
          pp.keys.push_back(key);
        }
        if (mode == kFast32) {                         // tilings its device-built units can use
          const int g64 = r64_geom_for(m), gx = rx32_geom_for(m);
          pp.long64 |= m + 1 > kR64MaxW;
          pp.long32 |= m + 1 > kRX32MaxW;
          if (g64 >= 0) { pp.r64_geoms |= 1u << g64; pp.r64_pairs[g64] += nh; }
          if (gx >= 0) { pp.rx32_geoms |= 1u << gx; pp.rx32_pairs[gx] += nh; }
        }
        for (const LaneTemplate& t : tmpl) {
          StreamUnit su;
          su.read = (int)r;
          su.list = (int)(sh_out - ctx->shaps.data());
          su.cntA = (int)t.lanes[0].size(); su.cntB = (int)t.lanes[1].size();
          su.rowsA = t.rows[0]; su.rowsB = t.rows[1];
          su.ro = (int)roff[r];
          su.m = m;
          for (int ln = 0; ln < 2; ++ln)
            for (int h : t.lanes[ln])
              *sh_out++ = StreamHap{h, (int)(gid + (h - h0)), (int)hoff[h], (int)ctx->hap_len[h]};
          pp.su.push_back(su);
          pp.key.push_back((uint16_t)key);
          pp.key_rows[key] = std::max(pp.key_rows[key], std::max(t.rows[0], t.rows[1]));
        }
      }
    }
  };
  // parts: equal pair counts, a few per worker (large calls only)
  int nparts = 1;
  if (pool && N >= (1 << 16)) nparts = (int)std::min<int64_t>(B, 4 * (pool->size() + 1));
  trace.mark("offsets");
  std::vector<int64_t> pcut(nparts + 1, B);
  pcut[0] = 0;
  for (int i = 1, b = 0; i < nparts; ++i) {
    while (b < B && bgid[b + 1] <= N * i / nparts) ++b;
    pcut[i] = std::max<int64_t>(b, pcut[i - 1]);
  }
  std::vector<PlanPart> parts(nparts);
  if (nparts == 1) {
    plan_range(0, B, parts[0]);
  } else {
    std::function<void(int)> task = [&](int i) { plan_range(pcut[i], pcut[i + 1], parts[i]); };
    pool->run(nparts, task);
  }
  trace.mark("plan-parts");
  // merge in batch order: bins numbered by first appearance, units concatenated
  int64_t nunits_all = 0;
  for (const PlanPart& pp : parts) nunits_all += (int64_t)pp.su.size();
  ctx->su_all.resize(nunits_all);
  ctx->su_bin.resize(nunits_all);
  std::vector<int64_t> part_off(nparts + 1, 0);
  {
    int64_t o = 0;
    for (int ip = 0; ip < nparts; ++ip) {
      const PlanPart& pp = parts[ip];
      for (int key : pp.keys)
        if (sbin_index[key] < 0) {
          sbin_index[key] = (int)ctx->sbins.size();
          ctx->sbins.push_back(phmm_ctx::SBin{key / kMaxTilings, pp.key_geom[key], 0, 0});
        }
      for (int key : pp.keys)
        ctx->sbins[sbin_index[key]].max_rows = std::max(ctx->sbins[sbin_index[key]].max_rows, pp.key_rows[key]);
      part_off[ip] = o;
      o += (int64_t)pp.su.size();
      part_off[ip + 1] = o;
      for (int x = 0; x < kNumExactP; ++x) slot_pairs[x] += pp.slot_pairs[x];
      for (int g = 0; g < 8; ++g) { r64_pairs[g] += pp.r64_pairs[g]; rx32_pairs[g] += pp.rx32_pairs[g]; }
      long64 |= pp.long64; long32 |= pp.long32;
      stripe_pairs += pp.stripe_pairs;
      ctx->r64_geoms |= pp.r64_geoms; ctx->rx32_geoms |= pp.rx32_geoms;
      max_n = std::max(max_n, pp.max_n);
    }
  }
  // the parts' units and bin ids, concatenated in batch order (on the pool)
  auto copy_part = [&](int ip) {
    const PlanPart& pp = parts[ip];
    std::copy(pp.su.begin(), pp.su.end(), ctx->su_all.begin() + part_off[ip]);
    for (size_t i = 0; i < pp.key.size(); ++i) ctx->su_bin[part_off[ip] + i] = (uint8_t)sbin_index[pp.key[i]];
  };
  if (nparts == 1) {
    copy_part(0);
  } else {
    std::function<void(int)> task = copy_part;
    pool->run(nparts, task);
  }
  ctx->max_n = max_n;
  trace.mark("merge");
  // LPT order per tiling: one stable counting sort on (bin, descending lane rows), over the
  // parts in parallel (per-part histograms, key-major then part-ordered offsets)
  const int nsbins = (int)ctx->sbins.size();
  const int64_t nsunits = (int64_t)ctx->su_all.size();
  std::vector<int> bmax(nsbins, 0), bbase(nsbins + 1, 0);
  for (int bi = 0; bi < nsbins; ++bi) bmax[bi] = ctx->sbins[bi].max_rows;   // longest lane of the bin
  for (int bi = 0; bi < nsbins; ++bi) bbase[bi + 1] = bbase[bi] + bmax[bi] + 1;
  auto key = [&](int64_t i) {
    const StreamUnit& u = ctx->su_all[i];
    const int bi = ctx->su_bin[i];
    return bbase[bi] + bmax[bi] - std::max(u.rowsA, u.rowsB);
  };
  const int nkeys = bbase[nsbins];
  const int nsort = nparts == 1 ? 1 : std::min(nparts, pool->size() + 1);
  std::vector<int64_t> scut(nsort + 1);
  for (int i = 0; i <= nsort; ++i) scut[i] = nsunits * i / nsort;
  std::vector<std::vector<int64_t>> hist(nsort);
  auto count_part = [&](int ip) {
    hist[ip].assign(nkeys, 0);
    for (int64_t i = scut[ip]; i < scut[ip + 1]; ++i) ++hist[ip][key(i)];
  };
  if (nsort == 1) count_part(0);
  else { std::function<void(int)> task = count_part; pool->run(nsort, task); }
  ctx->su_cnt.assign(nkeys + 1, 0);           // su_cnt[k]: first slot of key k
  {
    int64_t o = 0;
    for (int k = 0; k < nkeys; ++k) {
      ctx->su_cnt[k] = (int)o;
      for (int ip = 0; ip < nsort; ++ip) {
        const int64_t c = hist[ip][k];
        hist[ip][k] = o;                        // this part's first slot for key k
        o += c;
      }
    }
    ctx->su_cnt[nkeys] = (int)o;
  }
  for (int bi = 0; bi < nsbins; ++bi) ctx->sbins[bi].dev_off = ctx->su_cnt[bbase[bi]];
  for (int bi = 0; bi < nsbins; ++bi)
    ctx->sbins[bi].count = (bi + 1 < nsbins ? ctx->su_cnt[bbase[bi + 1]] : nsunits) - ctx->sbins[bi].dev_off;
  ctx->h_sunits.resize(nsunits);
  auto scatter_part = [&](int ip) {
    for (int64_t i = scut[ip]; i < scut[ip + 1]; ++i) ctx->h_sunits[hist[ip][key(i)]++] = ctx->su_all[i];
  };
  if (nsort == 1) scatter_part(0);
  else { std::function<void(int)> task = scatter_part; pool->run(nsort, task); }
  // launch order of the concurrent tiling bins: largest total work first, so the small
  // bins fill the tails of the large ones
  {
    std::vector<double> work(nsbins, 0.0);
    for (int bi = 0; bi < nsbins; ++bi) {
      const StreamKernel& g = skern(ctx->sbins[bi].mode, ctx->sbins[bi].geom);
      for (int64_t i = ctx->sbins[bi].dev_off; i < ctx->sbins[bi].dev_off + ctx->sbins[bi].count; ++i) {
        const StreamUnit& u = ctx->h_sunits[i];
        work[bi] += (double)g.P * (g.K + 2.5) * (std::max(u.rowsA, u.rowsB) + g.P - 1) / g.P * g.P;
      }
    }
    ctx->sbin_order.resize(nsbins);
    std::iota(ctx->sbin_order.begin(), ctx->sbin_order.end(), 0);
    std::stable_sort(ctx->sbin_order.begin(), ctx->sbin_order.end(), [&](int a, int b) { return work[a] > work[b]; });
    if (trace.on) {                          // per bin: units, true cells, computed cells
      for (int bi = 0; bi < nsbins; ++bi) {
        const StreamKernel& g = skern(ctx->sbins[bi].mode, ctx->sbins[bi].geom);
        double tc = 0, cc = 0;
        for (int64_t i = ctx->sbins[bi].dev_off; i < ctx->sbins[bi].dev_off + ctx->sbins[bi].count; ++i) {
          const StreamUnit& u = ctx->h_sunits[i];
          const int64_t Q = (u.m + g.P * g.K) / (g.P * g.K);
          cc += 2.0 * Q * g.P * g.K * (std::max(u.rowsA, u.rowsB) + g.P - 1);
          tc += (double)u.m * (u.rowsA + u.rowsB);
        }
        fprintf(stderr, "[phmm bin] mode %d P %d K %d%s units %lld true %.4g computed %.4g\n", ctx->sbins[bi].mode, g.P,
                g.K, (ctx->sbins[bi].geom & kStripedBin) ? " striped" : "", (long long)ctx->sbins[bi].count, tc, cc);
      }
    }
  }
  trace.mark("units");
  auto t1 = std::chrono::steady_clock::now();
  ctx->plan_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();

  // ---- plan upload
  ctx->h_rmeta.resize(3 * R);
  std::copy(ctx->read_m.begin(), ctx->read_m.end(), ctx->h_rmeta.begin());
  std::copy(ctx->read_scale.begin(), ctx->read_scale.end(), ctx->h_rmeta.begin() + R);
  std::copy(read_ncap.begin(), read_ncap.end(), ctx->h_rmeta.begin() + 2 * R);
  CK(up(ctx->d_read_m, ctx->h_rmeta.data(), R));
  CK(up(ctx->d_read_scale, ctx->h_rmeta.data() + R, R));
  CK(up(ctx->d_read_ncap, ctx->h_rmeta.data() + 2 * R, R));
  CK(up(ctx->d_sunits, ctx->h_sunits.data(), ctx->h_sunits.size()));
  CK(up(ctx->d_shaps, ctx->shaps.data(), ctx->shaps.size()));
  CK(ctx->d_gsum.ensure(R));
  CK(ctx->d_rflags.ensure(R));
  CK(ctx->d_acc.ensure(N));
  CK(ctx->d_status.ensure(N));
  CK(ctx->d_counters.ensure(kBinCounters + ctx->sbins.size()));
  // per-pair post-pass lists (device-appended): sized for every pair whose read maps there
  for (int s = 0; s < kNumExactP; ++s) {
    ctx->list_cap[s] = (int)std::max<int64_t>(slot_pairs[s], 1);
    CK(ctx->d_ex32[s].ensure(ctx->list_cap[s]));
    CK(ctx->d_ex64[s].ensure(ctx->list_cap[s]));
    CK(ctx->d_fx64[s].ensure(ctx->list_cap[s]));
  }
  // Boundary-column scratch of the per-pair post-pass kernels (k_exact_all / k_fast64_all):
  // only their P = 32 slot stripes (reads >= 256), one sub-warp per warp, 2 buffers x
  // 3 values x (max_n + 1) rows each; the grid is capped so the scratch stays under
  // kColBudget even for very long haplotypes.
  {
    const size_t per_slot = 2 * 3 * (size_t)(max_n + 1);
    int max_m = 0;
    for (int64_t r = 0; r < R; ++r)
      if (ctx->read_cfg[r] >= 0) max_m = std::max(max_m, ctx->read_m[r]);
    const size_t per_cta = (size_t)(kThreads / 32) * per_slot * sizeof(double);
    ctx->post_grid = ctx->num_sms * 2;
    if (max_m + 1 > 32 * kExactK) {
      // a striped item runs on one warp (4 per CTA): more CTAs than ~items / 4 only add
      // scratch (a 100k-base haplotype: 19 MB of columns per CTA)
      const int64_t want = std::max<int64_t>(ctx->num_sms / 4, (stripe_pairs + 3) / 4);
      ctx->post_grid = (int)std::max<size_t>(1, std::min<size_t>({(size_t)ctx->post_grid, ctx->col_budget / per_cta,
                                                                 (size_t)want}));
      CK(ctx->d_cold.ensure((size_t)ctx->post_grid * (kThreads / 32) * per_slot));
    } else {
      CK(ctx->d_cold.ensure(1));       // never dereferenced: every post-pass read fits one stripe
    }
  }
  trace.mark("plan-upload");
  // content validation on the device (bases 0..4, qualities 0..93)
  CK(ctx->d_vflag.ensure(1));
  int* vflag = ctx->d_vflag.p;                 // also gates every kernel of the execute
  CK(cudaMemsetAsync(vflag, 0, sizeof(int), ctx->stream));
  if (RL + HL > 0) {
    const int64_t work = std::max<int64_t>(RL, HL) / 16 + 1;
    const int vblocks = (int)std::min<int64_t>(ctx->num_sms * 8, (work + 255) / 256);
    launch_validate(vblocks, ctx->stream, (const uint8_t*)ctx->d_rbases.p, ctx->d_bq.p, ctx->d_iq.p, ctx->d_dq.p,
                    ctx->d_gq.p, RL, (const uint8_t*)ctx->d_hbases.p, HL, vflag);
    CK(cudaGetLastError());
  }
  CK(cudaMemcpyAsync(ctx->h_vflag, vflag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaEventRecord(ctx->ev_up1, ctx->stream));
  ctx->h2d_bytes = bytes;
  ctx->h2d_ms = 0.0;
  if (!ctx->async) {
    int rc = check_validation(ctx);
    if (rc != PHMM_SUCCESS) return rc;
    float h2d = 0.f;
    cudaEventElapsedTime(&h2d, ctx->ev_up0, ctx->ev_up1);
    ctx->h2d_ms = h2d;
  }

  // device-built stream units (FP64 retries, exact guard-band reruns): sized for every
  // pair of the FP32 stream units (worst case: all of them)
  int64_t streamed = 0;
  for (auto& sb : ctx->sbins)
    if (sb.mode == kFast32)
      for (int64_t i = sb.dev_off; i < sb.dev_off + sb.count; ++i)
        streamed += ctx->h_sunits[i].cntA + ctx->h_sunits[i].cntB;
  const bool r64 = (opt->flags & PHMM_FLAG_RETRY_F64) && streamed > 0 && ctx->r64_geoms;
  const bool rx32 = streamed > 0 && ctx->rx32_geoms;
  if (!r64) ctx->r64_geoms = 0;
  if (!rx32) ctx->rx32_geoms = 0;
  // second-stage FP64 units (r64b: guard-band pairs whose exact rerun underflows, from the
  // exact-FP32 stream units, the inline reruns and the per-pair exact list) live in a
  // second region of the FP64 unit list of their tiling, for every tiling: per-pair FP64 is
  // latency bound (c5 5.4 ms for 53k pairs) and rounds differently from the stream kernel,
  // so with one FP64 kernel for all retries a pair's value does not depend on the path
  // (or the chunking) that reran it
  const bool longer = streamed >= kMidCallPairs;   // longer device-built retry units
  const unsigned r64b_geoms = r64 ? ctx->r64_geoms : 0u;
  for (int g = 0; g < kNumR64Geoms; ++g)
    if (ctx->r64_geoms & (1u << g))
      CK(ctx->d_r64u[g].ensure(r64_pairs[g] * ((r64b_geoms >> g) & 1 ? 2 : 1)));
  for (int g = 0; g < kNumRX32Geoms; ++g)
    if (ctx->rx32_geoms & (1u << g)) CK(ctx->d_rx32u[g].ensure(rx32_pairs[g]));
  if (r64) CK(ctx->d_r64h.ensure(streamed));
  if (rx32) CK(ctx->d_rx32h.ensure(streamed));
  EngineDev& E = ctx->dev;
  E.rbases = ctx->d_rbases.p; E.bq = ctx->d_bq.p; E.iq = ctx->d_iq.p; E.dq = ctx->d_dq.p; E.gq = ctx->d_gq.p;
  E.roff = ctx->d_roff.p; E.hbases = ctx->d_hbases.p; E.hoff = ctx->d_hoff.p;
  E.read_m = ctx->d_read_m.p; E.read_scale = ctx->d_read_scale.p; E.read_ncap = ctx->d_read_ncap.p;
  E.read_gsum = ctx->d_gsum.p; E.read_flags = ctx->d_rflags.p; E.lut = ctx->d_lut.p;
  E.acc = ctx->d_acc.p; E.status = ctx->d_status.p;
  E.invalid = ctx->d_vflag.p;
  for (int s = 0; s < kNumExactP; ++s) {
    E.ex32[s] = ctx->d_ex32[s].p; E.ex64[s] = ctx->d_ex64[s].p; E.fx64[s] = ctx->d_fx64[s].p;
  }
  E.fx64_count = ctx->d_counters.p + 20;
  E.ex32_count = ctx->d_counters.p + 0;
  E.ex64_count = ctx->d_counters.p + kNumExactP;
  for (int s = 0; s < kNumExactP; ++s) E.list_cap[s] = ctx->list_cap[s];
  E.retry_f64 = (opt->flags & PHMM_FLAG_RETRY_F64) ? 1 : 0;
  E.band_inline = ctx->d_counters.p + 16;
  // inline guard-band reruns are slow per pair (scalar exact recursion inside an FP32
  // warp): a budget per call, split between the chunk contexts of a pipelined call
  static const int band_pct = [] {              // experiments: PHMM_BAND_INLINE (% of #SM per launch)
    const char* e = getenv("PHMM_BAND_INLINE");
    return e ? std::max(0, atoi(e)) : 50;       // c3 -1..2 %, c2 unchanged (was 200)
  }();
  E.band_budget = band_pct * ctx->num_sms / 100 / std::max(1, ctx->budget_div);
  // tilings that cannot get work (no streamed read of that width) stay null
  auto lists = [&](RetryLists& L, DBuf<StreamUnit>* u, int ng, DBuf<StreamHap>& h, unsigned geoms, int base,
                   const int64_t* gpairs) {
    for (int g = 0; g < 8; ++g) L.units[g] = (g < ng && (geoms & (1u << g))) ? u[g].p : nullptr;
    L.enabled = geoms ? 1 : 0;
    L.haps = geoms ? h.p : nullptr;
    L.count = ctx->d_counters.p + base;
    L.hap_count = ctx->d_counters.p + base + 8;
    L.overflow = ctx->d_counters.p + base + 9;
    for (int g = 0; g < 8; ++g) L.unit_cap[g] = (g < ng && (geoms & (1u << g))) ? (int)gpairs[g] : 0;
    L.hap_cap = geoms ? (int)streamed : 0;
    // short units keep small post-pass lists parallel (their size is unknown when the
    // grid is sized); large calls get longer units (less fill/drain and setup per pair)
    // (FP64 / exact lane haplotypes: c5 8 / 5 250.7 ms < 4 / 5 252.4 < 4 / 3 252.9 < 3 / 3
    // 257.6; 512k pairs 8 / 5 13.5 ms < 4 / 3 13.6 < 2 / 1 13.9; c3 (65k) equal)
    L.lane_haps = &L == &E.r64 ? (longer ? 8 : kRetryLaneHaps64) : (longer ? 5 : kRetryLaneHapsX32);
  };
  lists(E.r64, ctx->d_r64u, kNumR64Geoms, ctx->d_r64h, ctx->r64_geoms, kCtrR64, r64_pairs);
  lists(E.rx32, ctx->d_rx32u, kNumRX32Geoms, ctx->d_rx32h, ctx->rx32_geoms, kCtrRX32, rx32_pairs);
  // second stage: guard-band pairs whose exact rerun underflows get FP64 stream units in
  // the upper half of their tiling's FP64 list (haplotype entries share the first stage's
  // array: the two sets of pairs are disjoint), run after the post-pass instead of the
  // per-pair kernel
  {
    E.r64b = E.r64;
    for (int x = 0; x < 8; ++x) E.r64b.units[x] = nullptr;
    E.r64b.count = ctx->d_counters.p + kCtrR64b;
    E.r64b.lane_haps = longer ? E.r64.lane_haps : 1;
    E.r64b.enabled = r64b_geoms ? 1 : 0;
    for (int g = 0; g < kNumR64Geoms; ++g)
      if ((r64b_geoms >> g) & 1) E.r64b.units[g] = ctx->d_r64u[g].p + r64_pairs[g];
  }
  // grids of the stream launches, and boundary-column space for the ones that can meet
  // striped units (reads longer than the tiling width): per sub-warp slot 2 columns x
  // 3 states x (longest lane + 2) two-lane values.  A grid whose columns would exceed
  // kColBudget (very long haplotypes) is shrunk to fit.
  {
    int64_t col_total = 0;
    auto col_per_cta = [&](int mode, const StreamKernel& K, int max_rows) -> int64_t {
      const int64_t v = (mode == kFast64 || mode == kExact64) ? 16 : 8;
      return (int64_t)4 * (32 / K.P) * 6 * col_rows_for(K.P, max_rows) * v;
    };
    auto fit = [&](int grid, int64_t per_cta) {
      return (int)std::max<int64_t>(1, std::min<int64_t>(grid, (int64_t)ctx->col_budget / per_cta));
    };
    for (auto& sb : ctx->sbins) {
      const StreamKernel& K = skern(sb.mode, sb.geom);
      const int G = 32 / K.P;
      const int64_t groups = (sb.count + G - 1) / G;
      const bool striped = (sb.geom & kStripedBin) != 0;
      // striped bins with few units run in team mode (a CTA per unit): one CTA per unit
      const int64_t want = striped && groups * 2 <= (int64_t)ctx->num_sms * K.occ * 4 ? groups : (groups + 3) / 4;
      sb.grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->num_sms * occ_cap(K.occ), want));
      sb.col_off = striped ? col_total : -1;
      if (striped) {
        const int64_t per = col_per_cta(sb.mode, K, sb.max_rows);
        sb.grid = fit(sb.grid, per);
        col_total += sb.grid * per;
      }
    }
    // device-built units of striped reads: lanes of <= max(row capacity, longest haplotype)
    for (int g = 0; g < 8; ++g) { ctx->r64_col_off[g] = -1; ctx->rx32_col_off[g] = -1; }
    ctx->r64_grid = ctx->rx32_grid = 0;
    if (long64) {                                   // reads > 255 stripe on the widest FP64 tiling
      const int g = kNumR64Geoms - 1;
      if (ctx->r64_geoms & (1u << g)) {
        const StreamKernel& K = striped_tab(kFast64);
        const int64_t per = col_per_cta(kFast64, K, max_n);
        // every unit of the list holds >= 1 of its pairs: no more CTAs than that
        ctx->r64_grid = fit((int)std::min<int64_t>(ctx->num_sms * occ_cap(K.occ), std::max<int64_t>(1, r64_pairs[g])), per);
        ctx->r64_col_off[g] = col_total;
        col_total += ctx->r64_grid * per;
      }
    }
    if (long32) {                                   // reads > 511: exact FP32 stripes
      const int g = kNumRX32Geoms - 1;
      if (ctx->rx32_geoms & (1u << g)) {
        const StreamKernel& K = striped_tab(kExact32);
        const int64_t per = col_per_cta(kExact32, K, max_n);
        ctx->rx32_grid = fit((int)std::min<int64_t>(ctx->num_sms * occ_cap(K.occ), std::max<int64_t>(1, rx32_pairs[g])), per);
        ctx->rx32_col_off[g] = col_total;
        col_total += ctx->rx32_grid * per;
      }
    }
    if (col_total > 0) CK(ctx->d_colstream.ensure(col_total));
  }

  trace.mark("sync");
  trace.print("prepare");
  ctx->prepared = true;
  if (num_pairs_out) *num_pairs_out = N;
  return PHMM_SUCCESS;
}

// CUDA-event timings of a completed execute: whole, FP32 stream phase, and the four phases
static int record_timing(phmm_ctx* ctx) {
  float dev = 0.f, fast = 0.f, ph[4] = {0.f, 0.f, 0.f, 0.f};
  CK(cudaEventElapsedTime(&dev, ctx->ev_start, ctx->ev_end));
  CK(cudaEventElapsedTime(&fast, ctx->ev_fast0, ctx->ev_fast1));
  CK(cudaEventElapsedTime(&ph[0], ctx->ev_start, ctx->ev_fast0));
  CK(cudaEventElapsedTime(&ph[2], ctx->ev_fast1, ctx->ev_post1));
  CK(cudaEventElapsedTime(&ph[3], ctx->ev_post1, ctx->ev_end));
  ph[1] = fast;
  ctx->last_dev_ms = dev;
  ctx->last_fast_ms = fast;
  for (int i = 0; i < 4; ++i) ctx->last_phase_ms[i] = ph[i];
  if (getenv("PHMM_TRACE")) {                 // post-pass list sizes (device-appended)
    int c[kBinCounters];
    if (cudaMemcpy(c, ctx->d_counters.p, sizeof(c), cudaMemcpyDeviceToHost) == cudaSuccess) {
      int r64 = 0, rx32 = 0;
      for (int g = 0; g < 8; ++g) { r64 += c[kCtrR64 + g]; rx32 += c[kCtrRX32 + g]; }
      fprintf(stderr, "[phmm lists] per-pair ex32 %d %d %d %d | ex64 %d %d %d %d | fx64 %d %d %d %d | "
                      "stream units r64 %d (entries %d) rx32 %d (entries %d)\n",
              c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7], c[20], c[21], c[22], c[23], r64, c[kCtrR64 + 8],
              rx32, c[kCtrRX32 + 8]);
    }
  }
  return PHMM_SUCCESS;
}

int phmm_execute(phmm_ctx* ctx) {
  if (!ctx) return PHMM_ERR_INVALID;
  if (!ctx->prepared) return ctx->fail(PHMM_ERR_STATE, "phmm_execute before phmm_prepare");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const EngineDev& E = ctx->dev;
  const int64_t N = ctx->num_pairs;
  int launches = 0;
  CK(cudaEventRecord(ctx->ev_start, st));
  const int nsb = (int)ctx->sbins.size();
  int* bin_ctr = ctx->d_counters.p + kBinCounters;
  // the work counters and per-pair status are reset by k_precompute itself: no small
  // H2D copy / memsets on the critical path
  // L2 prefetch of the per-unit inputs on a side stream, beside k_precompute (joined with
  // the FP32 phase; the bench flushes L2 between steps)
  CK(cudaEventRecord(ctx->ev_pre, st));
  CK(cudaStreamWaitEvent(ctx->aux[phmm_ctx::kAux - 1], ctx->ev_pre, 0));
  launch_l2_prefetch(ctx->num_sms * 2, ctx->aux[phmm_ctx::kAux - 1], ctx->d_sunits.p,
                     (int64_t)ctx->h_sunits.size() * (int64_t)sizeof(StreamUnit), ctx->d_shaps.p,
                     (int64_t)ctx->shaps.size() * (int64_t)sizeof(StreamHap), ctx->d_hbases.p, ctx->hap_bytes,
                     ctx->d_rbases.p, ctx->d_bq.p, ctx->read_bytes);
  ++launches;
  launch_precompute(ctx->num_reads, st, E, ctx->d_counters.p, kBinCounters + nsb, N);
  ++launches;
  CK(cudaEventRecord(ctx->ev_pre, st));
  CK(cudaEventRecord(ctx->ev_fast0, st));
  // Stream bins (one persistent launch per tiling) go round-robin onto side streams so a
  // bin's tail (its last CTAs draining) overlaps the next bin's work.
  constexpr int kStreamAux = phmm_ctx::kAux - 1;
  int nlaunch = 0;
  auto side = [&](int i) -> cudaStream_t { return ctx->aux[i % kStreamAux]; };
  bool used[phmm_ctx::kAux] = {};
#define CKE(call) do { cudaError_t _e = (call); if (_e != cudaSuccess) return _e; } while (0)
  auto fork = [&]() -> cudaError_t {
    CKE(cudaEventRecord(ctx->ev_pre, st));
    for (int a = 0; a < phmm_ctx::kAux; ++a) {
      used[a] = false;
      CKE(cudaStreamWaitEvent(ctx->aux[a], ctx->ev_pre, 0));
    }
    return cudaSuccess;
  };
  auto join = [&]() -> cudaError_t {
    for (int a = 0; a < phmm_ctx::kAux; ++a) {
      if (!used[a]) continue;
      CKE(cudaEventRecord(ctx->ev_join[a], ctx->aux[a]));
      CKE(cudaStreamWaitEvent(st, ctx->ev_join[a], 0));
    }
    return cudaSuccess;
  };
#undef CKE
  CK(fork());
  used[phmm_ctx::kAux - 1] = true;                 // joins the L2 prefetch as well
  for (int oi = 0; oi < nsb; ++oi) {
    const int bi = ctx->sbin_order[oi];             // costliest tiling first
    const auto& sb = ctx->sbins[bi];
    const int nu = (int)sb.count;
    if (nu == 0) continue;
    const StreamKernel& SKn = skern(sb.mode, sb.geom);
    used[nlaunch % kStreamAux] = true;
    SKn.launch(dim3(sb.grid), SKn.smem, side(nlaunch++), E, ctx->d_sunits.p + sb.dev_off, ctx->d_shaps.p, nu, nullptr,
               bin_ctr + bi, sb.col_off >= 0 ? ctx->d_colstream.p + sb.col_off : nullptr,
               col_rows_for(SKn.P, sb.max_rows));
    ++launches;
  }
  CK(join());
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev_fast1, st));
  // Post-pass.  (a) concurrently: device-built stream units -- bit-exact FP32 reruns of
  // guard-band pairs and FP64 retries of FP32-underflowed pairs -- and the per-pair exact
  // FP32 list; (b) per-pair FP64 retries (fed by (a)); (c) per-pair bit-exact FP64 (fed by
  // everything before).  Only tilings some streamed read can use are launched.
  CK(fork());
  used[0] = true;
  launch_exact_all_f32(ctx->post_grid, ctx->aux[0], E, ctx->d_counters.p + 8, (float*)ctx->d_cold.p, ctx->max_n + 1);
  ++launches;
  int nside = 0;
  auto post = [&](const StreamKernel& SKn, const RetryLists& L, int g, int* work, int64_t col_off, int grid) {
    const int a = 1 + (nside++ % (phmm_ctx::kAux - 1));
    used[a] = true;
    SKn.launch(dim3(grid), SKn.smem, ctx->aux[a], E, L.units[g], L.haps, L.unit_cap[g], L.count + g, work,
               col_off >= 0 ? ctx->d_colstream.p + col_off : nullptr, col_rows_for(SKn.P, ctx->max_n));
    ++launches;
    return a;
  };
  for (int g = kNumR64Geoms - 1; g >= 0; --g)
    if (ctx->r64_geoms & (1u << g)) {
      const bool str = ctx->r64_col_off[g] >= 0;
      const StreamKernel& SKn = str ? striped_tab(kFast64) : stream_table_fast64()[g];
      post(SKn, E.r64, g, ctx->d_counters.p + kCtrR64Work + g, ctx->r64_col_off[g],
           str ? ctx->r64_grid : ctx->num_sms * occ_cap(SKn.occ));
    }
  bool x32_on[phmm_ctx::kAux] = {};
  for (int g = kNumRX32Geoms - 1; g >= 0; --g)
    if (ctx->rx32_geoms & (1u << g)) {
      const bool str = ctx->rx32_col_off[g] >= 0;
      const StreamKernel& SKn = str ? striped_tab(kExact32) : stream_table_exact32()[g];
      x32_on[post(SKn, E.rx32, g, ctx->d_counters.p + kCtrRX32Work + g, ctx->rx32_col_off[g],
                  str ? ctx->rx32_grid : ctx->num_sms * occ_cap(SKn.occ))] = true;
    }
  // second-stage FP64 units (guard-band pairs whose exact rerun underflowed) depend only on
  // the exact-FP32 kernels (stream units, and the per-pair list on aux[0]; the inline reruns
  // ran in the FP32 phase): single-stripe tilings start, one stream each, as soon as those
  // are done, beside the first-stage FP64 units (c5: their 3-4 ms tail overlapped); striped
  // ones share their tiling's boundary columns with the first stage and run after it
  x32_on[0] = true;
  bool r64b_side = false;
  for (int g = 0; g < kNumR64Geoms; ++g) r64b_side |= E.r64b.units[g] && ctx->r64_col_off[g] < 0;
  if (r64b_side)
    for (int x = 0; x < phmm_ctx::kAux; ++x)
      if (x32_on[x]) CK(cudaEventRecord(ctx->ev_x32[x], ctx->aux[x]));
  bool r64b_on[kNumR64Geoms] = {};
  for (int g = kNumR64Geoms - 1; g >= 0 && r64b_side; --g) {
    if (!E.r64b.units[g] || ctx->r64_col_off[g] >= 0) continue;
    cudaStream_t b = ctx->r64b_st[g];
    for (int x = 0; x < phmm_ctx::kAux; ++x)
      if (x32_on[x]) CK(cudaStreamWaitEvent(b, ctx->ev_x32[x], 0));
    const StreamKernel& SKn = stream_table_fast64()[g];
    SKn.launch(dim3(ctx->num_sms * occ_cap(SKn.occ)), SKn.smem, b, E, E.r64b.units[g], E.r64b.haps,
               E.r64b.unit_cap[g], E.r64b.count + g, ctx->d_counters.p + kCtrR64bWork + g, nullptr,
               col_rows_for(SKn.P, ctx->max_n));
    ++launches;
    CK(cudaEventRecord(ctx->ev_r64b[g], b));
    r64b_on[g] = true;
  }
  CK(join());
  for (int g = 0; g < kNumR64Geoms; ++g)
    if (r64b_on[g]) CK(cudaStreamWaitEvent(st, ctx->ev_r64b[g], 0));
  CK(cudaEventRecord(ctx->ev_post1, st));
  for (int g = kNumR64Geoms - 1; g >= 0; --g) {   // striped second-stage units
    if (!E.r64b.units[g] || ctx->r64_col_off[g] < 0) continue;
    const bool str = ctx->r64_col_off[g] >= 0;
    const StreamKernel& SKn = str ? striped_tab(kFast64) : stream_table_fast64()[g];
    SKn.launch(dim3(str ? ctx->r64_grid : ctx->num_sms * occ_cap(SKn.occ)), SKn.smem, st, E, E.r64b.units[g],
               E.r64b.haps, E.r64b.unit_cap[g], E.r64b.count + g, ctx->d_counters.p + kCtrR64bWork + g,
               str ? ctx->d_colstream.p + ctx->r64_col_off[g] : nullptr, col_rows_for(SKn.P, ctx->max_n));
    ++launches;
  }
  if (ctx->flags & PHMM_FLAG_RETRY_F64) {
    launch_fast64_all(ctx->post_grid, st, E, ctx->d_counters.p + 24, ctx->d_cold.p, ctx->max_n + 1);
    ++launches;
  }
  launch_exact_all_f64(ctx->post_grid, st, E, ctx->d_counters.p + 12, ctx->d_cold.p, ctx->max_n + 1);
  ++launches;
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev_end, st));
  ctx->last_launches = launches;
  ctx->executed = true;
  if (ctx->async) return PHMM_SUCCESS;
  CK(cudaEventSynchronize(ctx->ev_end));
  return record_timing(ctx);
}

// D2H of the raw results into pinned staging, asynchronous on the engine stream
static int fetch_enqueue(phmm_ctx* ctx) {
  const int64_t N = ctx->num_pairs;
  if (N > ctx->h_res_cap) {                 // pinned staging for the D2H of acc + status
    if (ctx->h_acc) cudaFreeHost(ctx->h_acc);
    if (ctx->h_st) cudaFreeHost(ctx->h_st);
    ctx->h_acc = nullptr; ctx->h_st = nullptr; ctx->h_res_cap = 0;
    CK(cudaMallocHost(&ctx->h_acc, N * sizeof(double)));
    CK(cudaMallocHost(&ctx->h_st, N));
    ctx->h_res_cap = N;
  }
  CK(cudaEventRecord(ctx->ev_d0, ctx->stream));
  if (N > 0) {
    CK(cudaMemcpyAsync(ctx->h_acc, ctx->d_acc.p, N * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(ctx->h_st, ctx->d_status.p, N, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaEventRecord(ctx->ev_d1, ctx->stream));
  return PHMM_SUCCESS;
}

static int fetch_complete(phmm_ctx* ctx, double* out_log10, uint8_t* out_status, phmm_stats* stats);

int phmm_fetch(phmm_ctx* ctx, double* out_log10, uint8_t* out_status, phmm_stats* stats) {
  if (!ctx) return PHMM_ERR_INVALID;
  if (!ctx->executed) return ctx->fail(PHMM_ERR_STATE, "phmm_fetch before phmm_execute");
  CK(cudaSetDevice(ctx->device));
  int rc = fetch_enqueue(ctx);
  if (rc != PHMM_SUCCESS) return rc;
  return fetch_complete(ctx, out_log10, out_status, stats);
}

static int fetch_complete(phmm_ctx* ctx, double* out_log10, uint8_t* out_status, phmm_stats* stats) {
  Trace trace;
  const int64_t N = ctx->num_pairs;
  const double* acc = ctx->h_acc;
  const uint8_t* st = ctx->h_st;
  CK(cudaEventSynchronize(ctx->ev_d1));
  float d2h = 0.f;
  cudaEventElapsedTime(&d2h, ctx->ev_d0, ctx->ev_d1);
  if (ctx->async) {            // chunk contexts: the execute / upload events completed by now
    float h2d = 0.f;
    record_timing(ctx);
    cudaEventElapsedTime(&h2d, ctx->ev_up0, ctx->ev_up1);
    ctx->h2d_ms = h2d;
  }
  // finishing (wavefront.py:428-434): host glibc log10 (= CPython math.log10), batches
  // split over a few threads
  struct Acc { int64_t cells = 0, fast = 0, exact = 0, f64 = 0, flagged = 0; };
  const int64_t B = ctx->num_batches;
  std::vector<int64_t> bgid(B + 1, 0);
  for (int64_t b = 0; b < B; ++b)
    bgid[b + 1] = bgid[b] + (ctx->batch_read_off[b + 1] - ctx->batch_read_off[b]) *
                                (ctx->batch_hap_off[b + 1] - ctx->batch_hap_off[b]);
  auto finish_range = [&](int64_t b0, int64_t b1, Acc* A) {
    for (int64_t b = b0; b < b1; ++b) {
      const int64_t r0 = ctx->batch_read_off[b], r1 = ctx->batch_read_off[b + 1];
      const int64_t h0 = ctx->batch_hap_off[b], h1 = ctx->batch_hap_off[b + 1];
      int64_t gid = bgid[b];
      for (int64_t r = r0; r < r1; ++r) {
        const int m = ctx->read_m[r];
        const int cfg = ctx->read_cfg[r];
        for (int64_t h = h0; h < h1; ++h, ++gid) {
          uint8_t s = st[gid];
          double v = NAN;
          if (cfg < 0) {
            s = PHMM_ST_CONFIG_TOO_SMALL;
          } else {
            const int kind = s & PHMM_ST_KIND_MASK;
            const bool retried = (s & PHMM_ST_RETRIED_F64) != 0;
            if (kind == PHMM_ST_OK) {
              const double a = acc[gid];
              if (a <= 0.0 || !std::isfinite(a)) {
                s = (uint8_t)((s & ~PHMM_ST_KIND_MASK) | PHMM_ST_NUMERIC_OVERFLOW);
              } else {
                const int scale = retried ? 0 : ctx->read_scale[r];
                v = std::log10(a) - scale * kLog10_2;
              }
            }
            const int k2 = s & PHMM_ST_KIND_MASK;
            if (k2 == PHMM_ST_OK || k2 == PHMM_ST_NUMERIC_OVERFLOW) A->cells += (int64_t)m * ctx->hap_len[h];
            if (k2 == PHMM_ST_OK) {
              if (retried) ++A->f64;
              else if (s & PHMM_ST_EXACT_F32) ++A->exact;
              else ++A->fast;
            }
            if (retried || k2 == PHMM_ST_NUMERIC_OVERFLOW) ++A->flagged;
          }
          if (out_log10) out_log10[gid] = v;
          if (out_status) out_status[gid] = s;
        }
      }
    }
  };
  trace.mark("d2h");
  phmm_ctx* owner = ctx->parent ? ctx->parent : ctx;    // chunk contexts share one pool
  if (!owner->pool && N >= 8192) {
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    owner->pool.reset(new WorkerPool(std::min(hw, kFinishThreads) - 1));
  }
  WorkerPool* pool = owner->pool.get();
  const int nth = pool ? (int)std::max<int64_t>(1, std::min<int64_t>(pool->size() + 1, N / 4096)) : 1;
  std::vector<Acc> parts(nth);
  if (nth == 1) {
    finish_range(0, B, &parts[0]);
  } else {
    std::vector<int64_t> cut(nth + 1, B);      // equal pair counts per task
    cut[0] = 0;
    int64_t b = 0;
    for (int i = 0; i < nth - 1; ++i) {
      const int64_t goal = N * (i + 1) / nth;
      while (b < B && bgid[b + 1] <= goal) ++b;
      cut[i + 1] = b;
    }
    std::function<void(int)> task = [&](int i) { finish_range(cut[i], cut[i + 1], &parts[i]); };
    pool->run(nth, task);
  }
  trace.mark("finish");
  trace.print("fetch");
  int64_t total_cells = 0, fast = 0, exact = 0, f64 = 0, flagged = 0;
  for (auto& A : parts) {
    total_cells += A.cells; fast += A.fast; exact += A.exact; f64 += A.f64; flagged += A.flagged;
  }
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    stats->num_pairs = N;
    stats->total_cells = total_cells;
    int64_t comp = 0;
    for (auto& sb : ctx->sbins) {
      const StreamKernel& g = skern(sb.mode, sb.geom);
      for (int64_t i = sb.dev_off; i < sb.dev_off + sb.count; ++i) {
        const StreamUnit& u = ctx->h_sunits[i];
        const int64_t Q = (u.m + g.P * g.K) / (g.P * g.K);
        comp += 2LL * Q * g.P * g.K * (std::max(u.rowsA, u.rowsB) + g.P - 1);
      }
    }
    stats->computed_cells = comp;
    stats->fast_pairs = fast;
    stats->exact_pairs = exact;
    stats->f64_pairs = f64;
    stats->flagged_pairs = flagged;
    stats->h2d_bytes = ctx->h2d_bytes;
    stats->d2h_bytes = N * (int64_t)(sizeof(double) + 1);
    stats->kernel_launches = ctx->last_launches;
    stats->device_ms = ctx->last_dev_ms;
    stats->fast_ms = ctx->last_fast_ms;
    stats->h2d_ms = ctx->h2d_ms;
    stats->d2h_ms = d2h;
    stats->plan_ms = ctx->plan_ms;
  }
  return PHMM_SUCCESS;
}

int phmm_last_timing(const phmm_ctx* ctx, double* device_ms, double* fast_ms, int* launches) {
  if (!ctx) return PHMM_ERR_INVALID;
  if (device_ms) *device_ms = ctx->last_dev_ms;
  if (fast_ms) *fast_ms = ctx->last_fast_ms;
  if (launches) *launches = ctx->last_launches;
  return PHMM_SUCCESS;
}

int phmm_last_phases(const phmm_ctx* ctx, double* phase_ms) {
  if (!ctx || !phase_ms) return PHMM_ERR_INVALID;
  for (int i = 0; i < 4; ++i) phase_ms[i] = ctx->last_phase_ms[i];
  return PHMM_SUCCESS;
}

int phmm_forward_matrices(phmm_ctx* ctx, const int8_t* read_bases, const uint8_t* base_qual,
                          const uint8_t* ins_qual, const uint8_t* del_qual, const uint8_t* gcp_qual, int32_t m,
                          const int8_t* hap_bases, int32_t n, int32_t scale_log2, double* M, double* I, double* D) {
  if (!ctx) return PHMM_ERR_INVALID;
  if (m < 1 || n < 1) return ctx->fail(PHMM_ERR_INVALID, "read and haplotype must contain at least one base");
  if (!read_bases || !base_qual || !ins_qual || !del_qual || !gcp_qual || !hap_bases || !M || !I || !D)
    return ctx->fail(PHMM_ERR_INVALID, "null argument");
  if ((int64_t)(m + 1) * (n + 1) > ((int64_t)1 << 28)) return ctx->fail(PHMM_ERR_INVALID, "matrices too large");
  for (int i = 0; i < m; ++i) {
    if ((uint8_t)read_bases[i] > 4) return ctx->fail(PHMM_ERR_INVALID, "base code outside A,C,G,T,N (0..4)");
    if (base_qual[i] > 93 || ins_qual[i] > 93 || del_qual[i] > 93 || gcp_qual[i] > 93)
      return ctx->fail(PHMM_ERR_INVALID, "quality values must be in [0, 93]");
  }
  for (int j = 0; j < n; ++j)
    if ((uint8_t)hap_bases[j] > 4) return ctx->fail(PHMM_ERR_INVALID, "base code outside A,C,G,T,N (0..4)");
  CK(cudaSetDevice(ctx->device));
  const size_t cells = (size_t)(m + 1) * (n + 1);
  const size_t in_bytes = 5 * (size_t)m + (size_t)n;
  unsigned char* d_in = nullptr;
  double* d_mat = nullptr;
  cudaError_t e = cudaMalloc(&d_in, in_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&d_mat, 3 * cells * sizeof(double));
  if (e == cudaSuccess) {
    const void* src[6] = {read_bases, base_qual, ins_qual, del_qual, gcp_qual, hap_bases};
    size_t off = 0;
    for (int x = 0; x < 6 && e == cudaSuccess; ++x) {
      const size_t len = x < 5 ? (size_t)m : (size_t)n;
      e = cudaMemcpyAsync(d_in + off, src[x], len, cudaMemcpyHostToDevice, ctx->stream);
      off += len;
    }
  }
  if (e == cudaSuccess) {
    // prob.py / reference.py:138: boundary 2.0 ** scale_log2 / n in f64
    const double boundary = ldexp(1.0, scale_log2) / (double)n;
    launch_matrices(ctx->stream, (const int8_t*)d_in, d_in + m, d_in + 2 * (size_t)m, d_in + 3 * (size_t)m,
                    d_in + 4 * (size_t)m, m, (const int8_t*)(d_in + 5 * (size_t)m), n, boundary, ctx->d_lut.p,
                    d_mat, d_mat + cells, d_mat + 2 * cells);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(M, d_mat, cells * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(I, d_mat + cells, cells * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(D, d_mat + 2 * cells, cells * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  if (d_in) cudaFree(d_in);
  if (d_mat) cudaFree(d_mat);
  if (e != cudaSuccess) return ctx->cuda_fail(e, "phmm_forward_matrices");
  return PHMM_SUCCESS;
}

int phmm_fast_geometry(int m, int n, int* P, int* K, int* Q) {
  if (m < 1 || n < 1 || !P || !K || !Q) return PHMM_ERR_INVALID;
  // the FP32 stream tiling a one-pair batch (m x n) is planned on
  const int g = choose_stream_geom(kFast32, m, n, n, INT64_MAX);
  const StreamKernel& k = g >= 0 ? stream_table_fast32()[g] : striped_fast32();
  *P = k.P; *K = k.K; *Q = (m + 1 + k.P * k.K - 1) / (k.P * k.K);
  return PHMM_SUCCESS;
}

// phmm_score pipelines large calls: the batches are cut into contiguous chunks (cut[c] ..
// cut[c+1]), each scored by one of `nctx` chunk contexts (device buffers, streams, pinned
// staging) used round-robin.  The host plans chunk c+1 while the GPU uploads and scores
// chunk c, and finishes chunk c while later chunks run; chunk kernels on separate streams
// also fill each other's tails.  A context is reused for chunk c + nctx only after chunk c
// is complete, so the device working set is bounded by nctx chunks (phmm_set_device_budget
// sizes the chunks for that).  Results are identical to the one-pass path (pairs are
// independent; gid order is batch-major, so a chunk owns a gid range).
static int score_chunked(phmm_ctx* ctx, const phmm_input* in, const phmm_options* opt, double* out_log10,
                         uint8_t* out_status, phmm_stats* stats, const std::vector<int64_t>& cut, int nctx,
                         size_t col_budget) {
  const int64_t B = in->num_batches;
  const int nchunks = (int)cut.size() - 1;
  std::vector<int64_t> pairs(B + 1, 0);
  for (int64_t b = 0; b < B; ++b)
    pairs[b + 1] = pairs[b] + (in->batch_read_off[b + 1] - in->batch_read_off[b]) *
                                  (in->batch_hap_off[b + 1] - in->batch_hap_off[b]);
  while ((int)ctx->chunks.size() < nctx) {
    phmm_ctx* c = new (std::nothrow) phmm_ctx();
    if (!c) return ctx->fail(PHMM_ERR_NOMEM, "chunk context");
    c->lut = ctx->lut;
    c->parent = ctx;
    ctx->chunks.push_back(c);
    const int rc = init_ctx(c, ctx->device);
    if (rc != PHMM_SUCCESS) return ctx->fail(rc, "chunk context: %s", c->err.c_str());
    c->async = true;
  }
  // on an error, chunks already enqueued are drained before returning (their contexts and
  // the caller's buffers must not be in use when the caller regains control)
  auto drain = [&]() {
    for (phmm_ctx* cx : ctx->chunks) {
      cudaStreamSynchronize(cx->stream);
      for (int a = 0; a < phmm_ctx::kAux; ++a) cudaStreamSynchronize(cx->aux[a]);
      for (int g = 0; g < kNumR64Geoms; ++g) cudaStreamSynchronize(cx->r64b_st[g]);
    }
  };
  phmm_stats total;
  memset(&total, 0, sizeof(total));
  // PHMM_TRACE=1: host timeline of the pipeline (ms since the call started)
  const bool tr = getenv("PHMM_TRACE") != nullptr;
  const auto tc0 = std::chrono::steady_clock::now();
  auto tnow = [&]() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tc0).count(); };
  float span = 0.f;                  // first chunk's execute start -> last execute end
  bool span_set = false;
  // complete chunk c: device validation verdict, then finishing into the caller's slice
  auto complete = [&](int c) -> int {
    if (cut[c + 1] <= cut[c]) return PHMM_SUCCESS;
    phmm_ctx* cx = ctx->chunks[c % nctx];
    const double tq = tnow();
    int rc = check_validation(cx);
    if (rc != PHMM_SUCCESS) return rc;
    phmm_stats cs;
    const int64_t g0 = pairs[cut[c]];
    rc = fetch_complete(cx, out_log10 ? out_log10 + g0 : nullptr, out_status ? out_status + g0 : nullptr, &cs);
    if (rc != PHMM_SUCCESS) return rc;
    float t = 0.f;
    if (span_set && cudaEventElapsedTime(&t, ctx->ev_span0, cx->ev_end) == cudaSuccess) span = std::max(span, t);
    total.fast_ms += cs.fast_ms;   // per-chunk FP32 phases (they overlap other chunks' work)
    total.h2d_ms += cs.h2d_ms;
    total.num_pairs += cs.num_pairs; total.total_cells += cs.total_cells;
    total.computed_cells += cs.computed_cells; total.fast_pairs += cs.fast_pairs;
    total.exact_pairs += cs.exact_pairs; total.f64_pairs += cs.f64_pairs;
    total.flagged_pairs += cs.flagged_pairs; total.h2d_bytes += cs.h2d_bytes; total.d2h_bytes += cs.d2h_bytes;
    total.kernel_launches += cs.kernel_launches; total.plan_ms += cs.plan_ms; total.d2h_ms += cs.d2h_ms;
    if (tr) fprintf(stderr, "[phmm chunk %d] complete %.2f -> %.2f ms (device %.2f ms)\n", c, tq, tnow(), cs.device_ms);
    return PHMM_SUCCESS;
  };
  for (int c = 0; c < nchunks; ++c) {
    phmm_ctx* cx = ctx->chunks[c % nctx];
    if (c >= nctx) {
      const int rc = complete(c - nctx);
      if (rc != PHMM_SUCCESS) {
        drain();
        return ctx->fail(rc, "%s", ctx->chunks[(c - nctx) % nctx]->err.c_str());
      }
    }
    const int64_t b0 = cut[c], b1 = cut[c + 1];
    if (b1 <= b0) continue;
    const int64_t r0 = in->batch_read_off[b0], r1 = in->batch_read_off[b1];
    const int64_t h0 = in->batch_hap_off[b0], h1 = in->batch_hap_off[b1];
    const int64_t ro0 = in->read_off[r0], ho0 = in->hap_off[h0];
    cx->c_roff.resize(r1 - r0 + 1);
    for (int64_t r = r0; r <= r1; ++r) cx->c_roff[r - r0] = in->read_off[r] - ro0;
    cx->c_hoff.resize(h1 - h0 + 1);
    for (int64_t h = h0; h <= h1; ++h) cx->c_hoff[h - h0] = in->hap_off[h] - ho0;
    cx->c_bro.resize(b1 - b0 + 1);
    cx->c_bho.resize(b1 - b0 + 1);
    for (int64_t b = b0; b <= b1; ++b) {
      cx->c_bro[b - b0] = in->batch_read_off[b] - r0;
      cx->c_bho[b - b0] = in->batch_hap_off[b] - h0;
    }
    phmm_input sub;
    sub.read_bases = in->read_bases + ro0;
    sub.base_qual = in->base_qual + ro0;
    sub.ins_qual = in->ins_qual + ro0;
    sub.del_qual = in->del_qual + ro0;
    sub.gcp_qual = in->gcp_qual + ro0;
    sub.read_off = cx->c_roff.data();
    sub.num_reads = r1 - r0;
    sub.hap_bases = in->hap_bases + ho0;
    sub.hap_off = cx->c_hoff.data();
    sub.num_haps = h1 - h0;
    sub.batch_read_off = cx->c_bro.data();
    sub.batch_hap_off = cx->c_bho.data();
    sub.num_batches = b1 - b0;
    int64_t n = 0;
    cx->budget_div = std::min(nchunks, nctx);
    cx->col_budget = col_budget;
    const double tp = tnow();
    int rc = phmm_prepare(cx, &sub, opt, &n);
    if (tr) fprintf(stderr, "[phmm chunk %d] prepare %.2f -> %.2f ms (%lld pairs)\n", c, tp, tnow(), (long long)n);
    if (rc == PHMM_SUCCESS && !span_set) {     // timing origin: the first execute's start
      rc = cudaEventRecord(ctx->ev_span0, cx->stream) == cudaSuccess ? PHMM_SUCCESS : PHMM_ERR_CUDA;
      span_set = rc == PHMM_SUCCESS;
    }
    if (rc == PHMM_SUCCESS) rc = phmm_execute(cx);
    if (rc == PHMM_SUCCESS) rc = fetch_enqueue(cx);
    if (rc != PHMM_SUCCESS) {
      drain();
      return ctx->fail(rc, "%s", cx->err.c_str());
    }
  }
  for (int c = std::max(0, nchunks - nctx); c < nchunks; ++c) {
    const int rc = complete(c);
    if (rc != PHMM_SUCCESS) {
      drain();
      return ctx->fail(rc, "%s", ctx->chunks[c % nctx]->err.c_str());
    }
  }
  if (tr) fprintf(stderr, "[phmm chunks] done %.2f ms\n", tnow());
  total.device_ms = span;
  ctx->last_dev_ms = span;
  ctx->last_fast_ms = (float)total.fast_ms;
  ctx->last_launches = total.kernel_launches;
  if (stats) *stats = total;
  return PHMM_SUCCESS;
}

// estimated device bytes of batch b in one prepare (see kDevBytesPerPair)
static int64_t batch_device_bytes(const phmm_input* in, int64_t b) {
  const int64_t r0 = in->batch_read_off[b], r1 = in->batch_read_off[b + 1];
  const int64_t h0 = in->batch_hap_off[b], h1 = in->batch_hap_off[b + 1];
  const int64_t rbytes = in->read_off[r1] - in->read_off[r0], hbytes = in->hap_off[h1] - in->hap_off[h0];
  return 5 * rbytes + hbytes + 48 * (r1 - r0) + 16 * (h1 - h0) + kDevBytesPerPair * (r1 - r0) * (h1 - h0);
}

// cut of the batches into contiguous chunks with pair counts proportional to w[0..nch)
static std::vector<int64_t> weighted_pair_cut(const phmm_input* in, const std::vector<int>& w) {
  const int64_t B = in->num_batches;
  const int nch = (int)w.size();
  std::vector<int64_t> pairs(B + 1, 0);
  for (int64_t b = 0; b < B; ++b)
    pairs[b + 1] = pairs[b] + (in->batch_read_off[b + 1] - in->batch_read_off[b]) *
                                  (in->batch_hap_off[b + 1] - in->batch_hap_off[b]);
  int64_t wsum = 0;
  for (int x : w) wsum += x;
  std::vector<int64_t> cut(nch + 1, B);
  cut[0] = 0;
  int64_t wacc = 0;
  for (int c = 1; c < nch; ++c) {
    wacc += w[c - 1];
    int64_t b = cut[c - 1];
    while (b < B && pairs[b] < pairs[B] * wacc / wsum) ++b;
    cut[c] = std::max(b, cut[c - 1]);
  }
  return cut;
}

int phmm_set_device_budget(phmm_ctx* ctx, int64_t bytes) {
  if (!ctx) return PHMM_ERR_INVALID;
  if (bytes < 0) return ctx->fail(PHMM_ERR_INVALID, "negative device budget");
  ctx->device_budget = bytes;
  return PHMM_SUCCESS;
}

int phmm_set_pipeline(phmm_ctx* ctx, int n) {
  if (!ctx) return PHMM_ERR_INVALID;
  if (n < 0 || n > kMaxScoreChunks) return ctx->fail(PHMM_ERR_INVALID, "pipeline depth %d not in 0..%d", n, kMaxScoreChunks);
  ctx->pipeline = n;
  return PHMM_SUCCESS;
}

int phmm_pin_host(void* ptr, int64_t bytes) {
  if (!ptr || bytes <= 0) return PHMM_ERR_INVALID;
  return cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterDefault) == cudaSuccess ? PHMM_SUCCESS : PHMM_ERR_CUDA;
}

int phmm_unpin_host(void* ptr) {
  if (!ptr) return PHMM_ERR_INVALID;
  return cudaHostUnregister(ptr) == cudaSuccess ? PHMM_SUCCESS : PHMM_ERR_CUDA;
}

int phmm_device_bytes(const phmm_ctx* ctx, int64_t* bytes) {
  if (!ctx || !bytes) return PHMM_ERR_INVALID;
  auto one = [](const phmm_ctx* c) -> int64_t {
    int64_t t = 0;
    auto add = [&](const auto& buf) { t += (int64_t)(buf.cap * sizeof(*buf.p)); };
    add(c->d_rbases); add(c->d_hbases); add(c->d_bq); add(c->d_iq); add(c->d_dq); add(c->d_gq);
    add(c->d_status); add(c->d_rflags); add(c->d_roff); add(c->d_hoff); add(c->d_read_m); add(c->d_read_scale);
    add(c->d_read_ncap); add(c->d_counters); add(c->d_vflag); add(c->d_gsum); add(c->d_lut); add(c->d_acc);
    add(c->d_sunits); add(c->d_shaps); add(c->d_r64h); add(c->d_rx32h); add(c->d_cold); add(c->d_colstream);
    for (int g = 0; g < kNumR64Geoms; ++g) add(c->d_r64u[g]);
    for (int g = 0; g < kNumRX32Geoms; ++g) add(c->d_rx32u[g]);
    for (int x = 0; x < kNumExactP; ++x) { add(c->d_ex32[x]); add(c->d_ex64[x]); add(c->d_fx64[x]); }
    return t;
  };
  int64_t t = one(ctx);
  for (const phmm_ctx* c : ctx->chunks) t += one(c);
  *bytes = t;
  return PHMM_SUCCESS;
}

int phmm_score(phmm_ctx* ctx, const phmm_input* in, const phmm_options* opt, double* out_log10,
               uint8_t* out_status, phmm_stats* stats) {
  if (!ctx) return PHMM_ERR_INVALID;
  Trace trace;
  const bool structure = in && opt && in->batch_read_off && in->batch_hap_off && in->read_off && in->hap_off &&
                         in->num_batches > 0;
  // validate the structure first (the chunk views index the offset arrays)
  int64_t pairs = 0;
  bool ok = structure && in->batch_read_off[0] == 0 && in->batch_hap_off[0] == 0 &&
            in->batch_read_off[in->num_batches] == in->num_reads && in->batch_hap_off[in->num_batches] == in->num_haps &&
            in->read_off[0] == 0 && in->hap_off[0] == 0;
  for (int64_t b = 0; ok && b < in->num_batches; ++b) {
    const int64_t nr = in->batch_read_off[b + 1] - in->batch_read_off[b];
    const int64_t nh = in->batch_hap_off[b + 1] - in->batch_hap_off[b];
    ok = nr > 0 && nh > 0;
    pairs += nr * nh;
  }
  // Device working-set bound: the caller's budget, or -- when the call would not fit the
  // free device memory -- half of that.  Over budget, the call streams through chunk
  // contexts reused round-robin, each chunk within budget / kBudgetCtx.
  constexpr int kBudgetCtx = 3;
  trace.mark("structure");
  if (ok) {
    int64_t budget = ctx->device_budget;
    int64_t est = 0;
    std::vector<int64_t> best(in->num_batches);
    for (int64_t b = 0; b < in->num_batches; ++b) est += (best[b] = batch_device_bytes(in, b));
    // (cudaMemGetInfo costs ~10 ms: only asked when the call is a sizeable part of HBM)
    if (budget == 0 && est > (int64_t)(ctx->total_mem / 8)) {
      size_t free_b = 0, total_b = 0;
      CK(cudaSetDevice(ctx->device));
      if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && est > (int64_t)(free_b * 0.6))
        budget = (int64_t)(free_b / 2);
    }
    if (budget > 0 && est > budget) {
      CK(cudaSetDevice(ctx->device));
      const int64_t per = std::max<int64_t>(1, budget / kBudgetCtx);
      std::vector<int64_t> cut{0};
      int64_t acc = 0;
      for (int64_t b = 0; b < in->num_batches; ++b) {
        if (acc > 0 && acc + best[b] > per) {
          cut.push_back(b);
          acc = 0;
        }
        acc += best[b];
      }
      cut.push_back(in->num_batches);
      const size_t col = (size_t)std::max<int64_t>(1 << 20, std::min<int64_t>(kColBudget, per / 8));
      return score_chunked(ctx, in, opt, out_log10, out_status, stats, cut,
                           std::min<int>(kBudgetCtx, (int)cut.size() - 1), col);
    }
  }
  trace.mark("budget");
  trace.print("score");
  // Pipelining (phmm_set_pipeline): large calls ramp -- the GPU idles while the first
  // chunk is planned and the host finishes the last one after the GPU is done, so both are
  // small (planning runs ~4x faster than the GPU scores, so chunk 1 is ready in time); the
  // middle chunks stay large (each chunk's phases end in a tail).  e2e per call
  // (tools/sweep_chunks_n8.sh): 1.25M pairs (the per-GPU share of c5 at N = 8) 1,5,1 38.0 ms
  // < 1,4,1 38.5 < 1,3,3,1 39.6 < 1,3,5,5,3,1 40.6 < one pass 52; 2.5M 1,6,1 / 1,5,1 72.7 <
  // 1,3,5,5,3,1 75.2; 5M 1,4,8,4,1 137.3 < 1,3,6,3,1 138.2 < 1,3,5,5,3,1 140.2 < 1,5,1 141;
  // c5 (10M) 1,4,8,8,4,1 267.7 < 1,4,8,4,1 268.5 < 1,3,5,5,3,1 270.2 < 1,6,6,1 276 < 1,8,1
  // 305; after the round's post-pass changes 1,5,10,10,5,1 260.3 < 1,6,14,14,6,1 260.6 <
  // 1,6,12,12,6,1 260.8 < 1,4,8,8,4,1 261.2 < 1,8,16,16,8,1 262.  Below 2^20 pairs one pass is as fast or faster (c2 2.1 vs 2.3+ ms chunked, c3
  // 3.8 vs 4.0+; tools/sweep_chunks_small2.sh).
  if (ok && ctx->pipeline != 1) {
    std::vector<int> w;
    if (ctx->pipeline > 1 && in->num_batches >= 2 * ctx->pipeline) w.assign(ctx->pipeline, 1);
    else if (ctx->pipeline == 0 && pairs >= 8000000) w = {1, 5, 10, 10, 5, 1};
    else if (ctx->pipeline == 0 && pairs >= 3500000) w = {1, 4, 8, 4, 1};
    else if (ctx->pipeline == 0 && pairs >= kBigCallPairs) w = {1, 5, 1};
    if (const char* env = getenv("PHMM_CHUNK_WEIGHTS"); env && !w.empty()) {   // experiments
      std::vector<int> ew;
      for (const char* p = env; *p;) {
        char* end = nullptr;
        const long v = strtol(p, &end, 10);
        if (end == p) break;
        if (v > 0) ew.push_back((int)v);
        p = *end ? end + 1 : end;
      }
      if (!ew.empty() && (int)ew.size() <= kMaxScoreChunks) w = ew;
    }
    if (!w.empty() && in->num_batches >= 2 * (int64_t)w.size()) {
      CK(cudaSetDevice(ctx->device));
      return score_chunked(ctx, in, opt, out_log10, out_status, stats, weighted_pair_cut(in, w), (int)w.size(),
                           kColBudget);
    }
  }
  int64_t n = 0;
  int rc = phmm_prepare(ctx, in, opt, &n);
  if (rc != PHMM_SUCCESS) return rc;
  rc = phmm_execute(ctx);
  if (rc != PHMM_SUCCESS) return rc;
  return phmm_fetch(ctx, out_log10, out_status, stats);
}

}  // extern "C"
