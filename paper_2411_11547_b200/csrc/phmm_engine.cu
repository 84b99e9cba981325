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
#include "phmm_kernels.cuh"

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

struct FastGeom { int P, K; };
// single-stripe widths W = P*K: 16 32 48 64 64 96 128 128 192 256 256 384 512
const FastGeom kFastGeoms[] = {{4, 4},  {4, 8},   {4, 12},  {4, 16},  {8, 8},   {8, 12}, {8, 16},
                               {16, 8}, {16, 12}, {16, 16}, {32, 8},  {32, 12}, {32, 16}};
constexpr int kNumFastGeoms = sizeof(kFastGeoms) / sizeof(kFastGeoms[0]);
constexpr int kExactP[kNumExactP] = {4, 8, 16, 32};
constexpr int kThreads = 128;
// device counters: [0,4) ex32 counts, [4,8) ex64 counts, [8,12) ex32 work, [12,16) ex64
// work, 16 inline guard-band pairs, [20,24) fx64 counts, [24,28) fx64 work, then the two
// device-built stream lists (counts[8], hap count, overflow) and their work counters,
// the validation flag (last slot), then one work counter per planned stream/legacy bin
constexpr int kCtrR64 = 32, kCtrRX32 = 44, kCtrR64Work = 56, kCtrRX32Work = 64;
constexpr int kCtrR64b = 72, kCtrR64bWork = 80;   // second-stage striped FP64 units: counts, work
constexpr int kBinCounters = 96;
constexpr int64_t kBigCallPairs = 1 << 20;   // device-built retry units grow above this          // fixed counter slots before the per-bin counters
constexpr int kFinishThreads = 16;        // host threads finishing log10 in phmm_fetch

struct Bin {
  int geom, Q;
  std::vector<FastUnit> units;
  int64_t dev_off = 0;     // offset into the device unit array
};

// fast-kernel launcher table: single-stripe and multi-stripe variant per geometry
template <int P, int K>
void launch_fast(dim3 g, size_t smem, cudaStream_t s, const EngineDev& E, const FastUnit* u, int nu,
                 int Q, int* ctr, float2* col, int rows) {
  if (Q > 1)
    k_fast<P, K, true><<<g, kThreads, smem, s>>>(E, u, nu, Q, ctr, col, rows);
  else
    k_fast<P, K, false><<<g, kThreads, smem, s>>>(E, u, nu, Q, ctr, col, rows);
}
typedef void (*FastLaunch)(dim3, size_t, cudaStream_t, const EngineDev&, const FastUnit*, int, int,
                           int*, float2*, int);
const FastLaunch kFastLaunch[kNumFastGeoms] = {
    launch_fast<4, 4>,  launch_fast<4, 8>,   launch_fast<4, 12>,  launch_fast<4, 16>, launch_fast<8, 8>,
    launch_fast<8, 12>, launch_fast<8, 16>,  launch_fast<16, 8>,  launch_fast<16, 12>,
    launch_fast<16, 16>, launch_fast<32, 8>, launch_fast<32, 12>, launch_fast<32, 16>};
const int kFastOcc[kNumFastGeoms] = {FastOcc<4>::value,  FastOcc<8>::value,  FastOcc<12>::value,
                                     FastOcc<16>::value, FastOcc<8>::value,  FastOcc<12>::value,
                                     FastOcc<16>::value, FastOcc<8>::value,  FastOcc<12>::value,
                                     FastOcc<16>::value, FastOcc<8>::value,  FastOcc<12>::value,
                                     FastOcc<16>::value};
#define FASTFN(P, K) (const void*)k_fast<P, K, false>, (const void*)k_fast<P, K, true>
const void* kFastFn[2 * kNumFastGeoms] = {FASTFN(4, 4),   FASTFN(4, 8),   FASTFN(4, 12), FASTFN(4, 16),
                                          FASTFN(8, 8),   FASTFN(8, 12),  FASTFN(8, 16), FASTFN(16, 8),
                                          FASTFN(16, 12), FASTFN(16, 16), FASTFN(32, 8), FASTFN(32, 12),
                                          FASTFN(32, 16)};
#undef FASTFN

// Streaming kernel family (single-stripe reads), one tiling table per mode
// (phmm_kernels.cuh: kFast32 / kFast64 / kExact32 / kExact64)
struct StreamKernel {
  int P, K, occ;
  size_t smem;
  const void* fn;
  void (*launch)(dim3, size_t, cudaStream_t, const EngineDev&, const StreamUnit*, const StreamHap*, int,
                 const int*, int*, void*, int);
};
template <int MODE, int P, int K, bool STRIPES>
void launch_stream_t(dim3 g, size_t smem, cudaStream_t s, const EngineDev& E, const StreamUnit* u,
                     const StreamHap* h, int nu, const int* nud, int* ctr, void* col, int col_rows) {
  k_stream<MODE, P, K, STRIPES><<<g, kThreads, smem, s>>>(E, u, h, nu, nud, ctr, col, col_rows);
}
template <int MODE, int P, int K, bool STRIPES = false>
StreamKernel SK() {
  const size_t elem = ModeOf<MODE>::F64 ? sizeof(double) : sizeof(float);   // 5*K*P entries per slot
  // striped instantiations add the boundary-column ring: per sub-warp slot 3 x kColRing
  // two-lane values
  return StreamKernel{P, K, STRIPES ? 2 : StreamOcc<MODE, K>::value,
                      96 * sizeof(double) + (size_t)4 * (32 / P) * 5 * K * P * elem + kStreamCodeBytesPerCta +
                          (STRIPES ? (size_t)4 * (32 / P) * 3 * kColRing * 2 * elem : 0),
                      (const void*)k_stream<MODE, P, K, STRIPES>, launch_stream_t<MODE, P, K, STRIPES>};
}
// kFast32: the k_fast tiling table (same order as kFastGeoms, so PHMM_FAST_GEOM applies),
// then K = 10, 14 tilings (2-wide emission chunks) for widths 80 .. 448
constexpr int kNumStreamFast32 = kNumFastGeoms + 6;
const StreamKernel kStreamFast32[kNumStreamFast32] = {
    SK<kFast32, 4, 4>(),   SK<kFast32, 4, 8>(),   SK<kFast32, 4, 12>(),  SK<kFast32, 4, 16>(),
    SK<kFast32, 8, 8>(),   SK<kFast32, 8, 12>(),  SK<kFast32, 8, 16>(),  SK<kFast32, 16, 8>(),
    SK<kFast32, 16, 12>(), SK<kFast32, 16, 16>(), SK<kFast32, 32, 8>(),  SK<kFast32, 32, 12>(),
    SK<kFast32, 32, 16>(), SK<kFast32, 8, 10>(),  SK<kFast32, 8, 14>(),  SK<kFast32, 16, 10>(),
    SK<kFast32, 16, 14>(), SK<kFast32, 32, 10>(), SK<kFast32, 32, 14>()};
// FP64 tilings, indexed by r64_geom_for(m): W = 32, 64, 96, 128, 192, 256
const StreamKernel kStreamFast64[kNumR64Geoms] = {SK<kFast64, 8, 4>(),  SK<kFast64, 16, 4>(),
                                                  SK<kFast64, 16, 6>(), SK<kFast64, 16, 8>(),
                                                  SK<kFast64, 32, 6>(), SK<kFast64, 32, 8>()};
const StreamKernel kStreamExact64[kNumR64Geoms] = {SK<kExact64, 8, 4>(),  SK<kExact64, 16, 4>(),
                                                   SK<kExact64, 16, 6>(), SK<kExact64, 16, 8>(),
                                                   SK<kExact64, 32, 6>(), SK<kExact64, 32, 8>()};
// exact FP32 tilings, indexed by rx32_geom_for(m): W = 32, 64, 96, 128, 192, 256, 384, 512
// (wide sub-warps: guard-band reruns are few and latency bound)
const StreamKernel kStreamExact32[kNumRX32Geoms] = {
    SK<kExact32, 8, 4>(),  SK<kExact32, 16, 4>(), SK<kExact32, 16, 6>(),  SK<kExact32, 32, 4>(),
    SK<kExact32, 32, 6>(), SK<kExact32, 32, 8>(), SK<kExact32, 32, 12>(), SK<kExact32, 32, 16>()};
const StreamKernel* const kStreamTab[4] = {kStreamFast32, kStreamFast64, kStreamExact32, kStreamExact64};
// reads longer than every tiling stripe over the widest one of their mode, in a separate
// instantiation (the column hand-off costs registers the single-stripe kernels keep)
const StreamKernel kStripedTab[4] = {SK<kFast32, 32, 16, true>(), SK<kFast64, 32, 8, true>(),
                                     SK<kExact32, 32, 8, true>(), SK<kExact64, 32, 8, true>()};
const int kStripedGeom[4] = {12, kNumR64Geoms - 1, kNumRX32Geoms - 1, kNumR64Geoms - 1};
const int kStreamTabN[4] = {kNumStreamFast32, kNumR64Geoms, kNumRX32Geoms, kNumR64Geoms};
constexpr int kMaxTilings = 24;
static_assert(kNumStreamFast32 <= kMaxTilings, "tiling table");

int stream_cap(int P) { return stream_cap_of(P); }

int exact_slot_host(int m) { return (m + 1 <= 32) ? 0 : (m + 1 <= 64) ? 1 : (m + 1 <= 128) ? 2 : 3; }

size_t fast_smem(int geom) {
  const FastGeom g = kFastGeoms[geom];
  return 96 * sizeof(double) + (size_t)(kThreads / 32) * (32 / g.P) * 5 * g.K * g.P * sizeof(float);
}
size_t exact_smem(int slot, size_t tsize) {
  const int P = kExactP[slot];
  return 96 * sizeof(double) + (size_t)(kThreads / 32) * (32 / P) * 5 * kExactK * P * tsize;
}

// Cost model for choosing a fast geometry: padded cells x (rows + fill/drain), plus a
// per-step overhead worth ~2.5 cells per thread.
// Single-stripe tilings (W >= m + 1) are preferred; reads longer than the widest tile
// (m >= 512) stripe over P = 32 tiles.
int forced_geom() {
  static int g = -2;
  if (g == -2) {
    g = -1;
    const char* env = getenv("PHMM_FAST_GEOM");      // tuning knob: "PxK"
    int P = 0, K = 0;
    if (env && sscanf(env, "%dx%d", &P, &K) == 2)
      for (int i = 0; i < kNumFastGeoms; ++i)
        if (kFastGeoms[i].P == P && kFastGeoms[i].K == K) g = i;
  }
  return g;
}

int choose_geom(int m, int nmax, int* Qout) {
  const int fg = forced_geom();
  if (fg >= 0) {
    const int W = kFastGeoms[fg].P * kFastGeoms[fg].K;
    *Qout = (m + 1 + W - 1) / W;
    return fg;
  }
  double best = 1e300;
  int bi = 0, bq = 1;
  const bool stripe = m + 1 > kFastGeoms[kNumFastGeoms - 1].P * kFastGeoms[kNumFastGeoms - 1].K;
  for (int g = 0; g < kNumFastGeoms; ++g) {
    const int P = kFastGeoms[g].P, K = kFastGeoms[g].K, W = P * K;
    const int Q = (m + 1 + W - 1) / W;
    if (stripe ? P != 32 : Q != 1) continue;
    const double cost = (double)Q * P * (K + 2.5) * (double)(nmax + P - 1);
    if (cost < best - 1e-9) { best = cost; bi = g; bq = Q; }
  }
  *Qout = bq;
  return bi;
}

// Streaming tiling for a read of length m whose batch has haplotype lengths summing to
// `total` (longest `nmax`): units of two lanes of ~total/2 rows, split when a lane would
// exceed the geometry's row-code capacity.  -1: no single-stripe streaming geometry.
// cost of streaming a read's haplotypes (total rows, longest nmax) on tiling g (1e300:
// infeasible or excluded by PHMM_FAST_GEOM)
// `lane_rows`: the call's lane-length budget (small calls split units further, below)
int64_t stream_geom_cost(int mode, int g, int64_t total, int nmax, int64_t lane_rows = INT64_MAX) {
  constexpr int64_t kInf = INT64_MAX;
  const int fg = forced_geom();
  if (mode == kFast32 && fg >= 0 && g != fg) return kInf;
  const int64_t P = kStreamTab[mode][g].P, K = kStreamTab[mode][g].K;
  if (nmax > stream_cap((int)P)) return kInf;
  const int64_t cap = std::min<int64_t>(stream_cap((int)P), std::max<int64_t>(nmax, lane_rows));
  const int64_t units = (total + 2 * cap - 1) / (2 * cap);
  const int64_t rows = std::min<int64_t>(cap, (total + 2 * units - 1) / (2 * units));
  return units * P * (2 * K + 5) * (rows + P - 1);     // 2 x (K + 2.5) per thread-row
}
int choose_stream_geom(int mode, int m, int64_t total, int nmax, int64_t lane_rows) {
  int64_t best = INT64_MAX;
  int bi = -1;
  for (int g = 0; g < kStreamTabN[mode]; ++g) {
    if (m + 1 > kStreamTab[mode][g].P * kStreamTab[mode][g].K) continue;
    const int64_t cost = stream_geom_cost(mode, g, total, nmax, lane_rows);
    if (cost < best) { best = cost; bi = g; }
  }
  return bi;
}
constexpr int kStripedBin = 1 << 10;          // geometry code of a striped bin
const StreamKernel& skern(int mode, int geom) {
  return (geom & kStripedBin) ? kStripedTab[mode] : kStreamTab[mode][geom];
}
// column rows a striped unit of tiling P can need (its row capacity + the row-0 slot)
int col_rows_for(int P) { return stream_cap_of(P) + 2; }
constexpr int kR64MaxW = 256, kRX32MaxW = 512;   // widest FP64 / exact-FP32 retry tilings

constexpr int kMaxScoreChunks = 8;
int score_chunks() {                          // phmm_score pipelining depth (PHMM_CHUNKS)
  static int v = -1;
  if (v < 0) {
    const char* env = getenv("PHMM_CHUNKS");
    v = env ? std::max(1, std::min(kMaxScoreChunks, atoi(env))) : 0;   // 0: by call size
  }
  return v;
}
constexpr int64_t kScoreChunkMinPairs = 32768;
bool score_chunking_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* env = getenv("PHMM_NO_CHUNK");
    v = (env && env[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

bool streaming_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* env = getenv("PHMM_NO_STREAM");
    v = (env && env[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

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
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_start = nullptr, ev_fast0 = nullptr, ev_fast1 = nullptr, ev_end = nullptr;
  cudaEvent_t ev_pre = nullptr;
  static constexpr int kAux = 8;              // side streams: kernels of a phase run concurrently
  cudaStream_t aux[kAux] = {};
  cudaEvent_t ev_join[kAux] = {};
  std::string err;
  std::vector<double> lut;

  // device buffers
  DBuf<int8_t> d_rbases, d_hbases;
  DBuf<uint8_t> d_bq, d_iq, d_dq, d_gq, d_status, d_rflags;
  DBuf<int64_t> d_roff, d_hoff;
  DBuf<int> d_read_m, d_read_scale, d_read_ncap, d_counters, d_vflag;
  DBuf<float> d_gsum;
  DBuf<double> d_lut, d_acc;
  DBuf<FastUnit> d_units;
  DBuf<StreamUnit> d_sunits;
  DBuf<StreamHap> d_shaps;
  DBuf<StreamUnit> d_r64u[kNumR64Geoms], d_rx32u[kNumRX32Geoms];
  DBuf<StreamHap> d_r64h, d_rx32h;
  DBuf<ExactItem> d_ex32[kNumExactP], d_ex64[kNumExactP], d_fx64[kNumExactP];
  DBuf<float2> d_colf;
  DBuf<double> d_cold;
  std::unique_ptr<WorkerPool> pool;         // host finishing threads (lazy)
  int* h_counts = nullptr;   // pinned: initial list counts (8) + zeros for work counters
  int* h_vflag = nullptr;    // pinned: device validation flag
  bool async = false;        // chunk contexts of phmm_score: no host syncs in prepare/execute
  phmm_ctx* parent = nullptr;
  int budget_div = 1;        // chunk contexts: number of chunks sharing the band budget
  std::vector<phmm_ctx*> chunks;             // chunk contexts (phmm_score pipelining), lazy
  std::vector<int64_t> c_roff, c_hoff, c_bro, c_bho;   // chunk views: rebased offsets
  double* h_acc = nullptr;   // pinned result staging (phmm_fetch)
  uint8_t* h_st = nullptr;
  int64_t h_res_cap = 0;

  // plan (host)
  bool prepared = false, executed = false;
  int64_t num_pairs = 0;
  int64_t num_reads = 0, num_haps = 0, num_batches = 0;
  std::vector<int64_t> batch_read_off, batch_hap_off, hap_len;
  std::vector<int> read_m, read_scale, read_cfg;   // read_cfg -1 = too small
  std::vector<Bin> bins;
  unsigned r64_geoms = 0, rx32_geoms = 0;   // device-built unit tilings that can get work
  struct SBin {
    int mode;
    int geom;
    int64_t count = 0;                      // units of this tiling
    int64_t dev_off = 0;                    // first unit in h_sunits / d_sunits
    int64_t col_off = -1;                   // striped units: column buffer (bytes), else -1
    int grid = 0;
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
  int host_ex32[kNumExactP] = {0, 0, 0, 0}, host_ex64[kNumExactP] = {0, 0, 0, 0};
  int max_n = 1;
  int flags = 0;
  int list_cap[kNumExactP] = {0, 0, 0, 0};
  int64_t h2d_bytes = 0;
  int64_t hap_bytes = 0, read_bytes = 0;
  double plan_ms = 0.0, h2d_ms = 0.0;
  int last_launches = 0;
  float last_dev_ms = 0.f, last_fast_ms = 0.f;
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
  CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ctx->ev_pre, cudaEventDisableTiming));
  for (int a = 0; a < phmm_ctx::kAux; ++a) {
    CK(cudaStreamCreateWithFlags(&ctx->aux[a], cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_join[a], cudaEventDisableTiming));
  }
  CK(cudaEventCreate(&ctx->ev_start));
  CK(cudaEventCreate(&ctx->ev_fast0));
  CK(cudaEventCreate(&ctx->ev_fast1));
  CK(cudaEventCreate(&ctx->ev_end));
  CK(cudaMallocHost(&ctx->h_counts, kBinCounters * sizeof(int)));
  CK(cudaMallocHost(&ctx->h_vflag, sizeof(int)));
  CK(ctx->d_lut.ensure(94));
  CK(cudaMemcpy(ctx->d_lut.p, ctx->lut.data(), 94 * sizeof(double), cudaMemcpyHostToDevice));
  for (int g = 0; g < 2 * kNumFastGeoms; ++g)
    CK(cudaFuncSetAttribute(kFastFn[g], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fast_smem(g / 2)));
  for (int md = 0; md < 4; ++md) {
    for (int g = 0; g < kStreamTabN[md]; ++g) {
      CK(cudaFuncSetAttribute(kStreamTab[md][g].fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)kStreamTab[md][g].smem));
      // one shared-memory carveout for every stream kernel: CTAs of different tilings can
      // share an SM without an L1/shared reconfiguration
      if (!getenv("PHMM_NO_CARVEOUT"))
        CK(cudaFuncSetAttribute(kStreamTab[md][g].fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    }
    CK(cudaFuncSetAttribute(kStripedTab[md].fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)kStripedTab[md].smem));
  }
  CK(cudaFuncSetAttribute((const void*)k_exact_all<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)exact_smem(0, 4)));
  CK(cudaFuncSetAttribute((const void*)k_exact_all<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)exact_smem(0, 8)));
  CK(cudaFuncSetAttribute((const void*)k_fast64_all, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)exact_smem(0, 8)));
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
  ctx->d_acc.release(); ctx->d_units.release(); ctx->d_sunits.release(); ctx->d_shaps.release();
  for (int g = 0; g < kNumR64Geoms; ++g) ctx->d_r64u[g].release();
  for (int g = 0; g < kNumRX32Geoms; ++g) ctx->d_rx32u[g].release();
  ctx->d_r64h.release();
  ctx->d_rx32h.release(); ctx->d_colf.release(); ctx->d_cold.release();
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
  if (ctx->ev_pre) cudaEventDestroy(ctx->ev_pre);
  for (int a = 0; a < phmm_ctx::kAux; ++a) {
    if (ctx->aux[a]) { cudaStreamSynchronize(ctx->aux[a]); cudaStreamDestroy(ctx->aux[a]); }
    if (ctx->ev_join[a]) cudaEventDestroy(ctx->ev_join[a]);
  }
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return PHMM_SUCCESS;
}

const char* phmm_last_error(const phmm_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

static int prepare_impl(phmm_ctx* ctx, const phmm_input* in, const phmm_options* opt, int64_t* num_pairs_out);

// waits for the prepare's uploads and the device content checks (k_validate)
static int check_validation(phmm_ctx* ctx) {
  CK(cudaEventSynchronize(ctx->ev_end));
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
  CK(cudaEventRecord(ctx->ev_start, ctx->stream));
  CK(up(ctx->d_rbases, in->read_bases, RL));
  CK(up(ctx->d_bq, in->base_qual, RL));
  CK(up(ctx->d_iq, in->ins_qual, RL));
  CK(up(ctx->d_dq, in->del_qual, RL));
  CK(up(ctx->d_gq, in->gcp_qual, RL));
  CK(up(ctx->d_roff, roff, R ? R + 1 : 0));
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
  int64_t memo_m = -1;
  int memo_cfg = -1;
  for (int64_t r = 0; r < R; ++r) {
    const int64_t m = roff[r + 1] - roff[r];
    if (m > (int64_t)1 << 30) return ctx->fail(PHMM_ERR_INVALID, "read too long");
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
  trace.mark("bind");
  // ---- pairs, hap pairing, units
  int64_t N = 0;
  for (int64_t b = 0; b < B; ++b)
    N += (ctx->batch_read_off[b + 1] - ctx->batch_read_off[b]) * (ctx->batch_hap_off[b + 1] - ctx->batch_hap_off[b]);
  if (N > INT32_MAX - 1) return ctx->fail(PHMM_ERR_INVALID, "too many pairs in one call (%lld)", (long long)N);
  ctx->num_pairs = N;
  const bool exact_mode = (opt->flags & PHMM_FLAG_EXACT) != 0;
  ctx->bins.clear();
  ctx->sbins.clear();
  ctx->r64_geoms = ctx->rx32_geoms = 0;
  ctx->su_all.clear();
  ctx->su_bin.clear();
  ctx->shaps.clear();
  // streaming units address reads/haplotypes with 32-bit offsets
  const bool use_stream = streaming_enabled() && RL < INT32_MAX && HL < INT32_MAX;
  std::vector<int> bin_index(kNumFastGeoms * 64, -1);
  int sbin_index[4 * kMaxTilings];
  std::fill(sbin_index, sbin_index + 4 * kMaxTilings, -1);
  std::vector<ExactItem> host32[kNumExactP], host64[kNumExactP];
  int64_t slot_pairs[kNumExactP] = {0, 0, 0, 0};
  int64_t r64_pairs[8] = {0}, rx32_pairs[8] = {0};
  bool long64 = false, long32 = false;          // streamed reads that stripe in the retry kernels
  int max_n = 1;
  int64_t gid = 0;
  std::vector<int> hidx;
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
  ModePlan mp[4];
  for (int md = 0; md < 4; ++md) {
    ModePlan& M = mp[md];
    M.n = kStreamTabN[md];
    for (int g = 0; g < M.n; ++g) M.wsort[g] = g;
    std::sort(M.wsort, M.wsort + M.n, [&](int x, int y) {
      return kStreamTab[md][x].P * kStreamTab[md][x].K < kStreamTab[md][y].P * kStreamTab[md][y].K;
    });
    for (int i = 0; i < M.n; ++i) M.wsorted[i] = kStreamTab[md][M.wsort[i]].P * kStreamTab[md][M.wsort[i]].K;
  }
  if (use_stream) ctx->shaps.reserve(N);
  // Lane budget: a call too small to fill the GPU with long lanes (few pairs, long
  // haplotypes: c4) splits its units until there are ~2 per sub-warp slot (#SM x 8 warps
  // x 2 sub-warps); latency, not per-unit overhead, bounds such calls.  Large calls keep
  // the row capacity as the only limit.
  int64_t lane_rows = INT64_MAX;
  {
    int64_t all_rows = 0;
    for (int64_t b = 0; b < B; ++b) {
      int64_t hs = 0;
      for (int64_t h = ctx->batch_hap_off[b]; h < ctx->batch_hap_off[b + 1]; ++h) hs += ctx->hap_len[h];
      all_rows += hs * (ctx->batch_read_off[b + 1] - ctx->batch_read_off[b]);
    }
    if (!getenv("PHMM_NO_LANE_BUDGET")) lane_rows = all_rows / (2 * 2 * (int64_t)ctx->num_sms * 16);
  }
  for (int64_t b = 0; b < B; ++b) {
    const int64_t r0 = ctx->batch_read_off[b], r1 = ctx->batch_read_off[b + 1];
    const int64_t h0 = ctx->batch_hap_off[b], h1 = ctx->batch_hap_off[b + 1];
    const int64_t nh = h1 - h0;
    int ncap = 1;
    int64_t batch_total = 0;
    for (int64_t h = h0; h < h1; ++h) {
      ncap = (int)std::max<int64_t>(ncap, ctx->hap_len[h]);
      batch_total += ctx->hap_len[h];
    }
    max_n = std::max(max_n, ncap);
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
      slot_pairs[exact_slot_host(m)] += nh;             // any pair may land in its slot's lists
      if (use_stream) {
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
          if (sg < 0 && m + 1 > M.wsorted[M.n - 1] &&   // longer than every tiling: stripes
              stream_geom_cost(mode, kStripedGeom[mode], batch_total, ncap) != INT64_MAX)
            sg = kStripedBin | kStripedGeom[mode];
          M.tmpl_geom = sg;
          const int ts = (sg & kStripedBin) ? kMaxTilings - 1 : sg;   // template cache slot
          if (sg >= 0 && !M.tvalid[ts]) {
            M.tvalid[ts] = true;
            std::vector<LaneTemplate>& tmpl = M.tmpls[ts];
            tmpl.clear();
            // greedy LPT over the length-sorted haplotypes: each to the lighter lane; a
            // new unit when a lane would exceed the tiling's row capacity or the call's
            // lane budget
            const int cap = (int)std::min<int64_t>(stream_cap(skern(mode, sg).P), std::max<int64_t>(lane_rows, 1));
            tmpl.emplace_back();
            for (int64_t x = 0; x < nh; ++x) {
              const int h = hidx[x];
              const int n = (int)ctx->hap_len[h];
              LaneTemplate* t = &tmpl.back();
              int ln = t->rows[0] <= t->rows[1] ? 0 : 1;
              if ((t->rows[ln] > 0 && t->rows[ln] + n > cap) || (int)t->lanes[ln].size() >= kStreamMaxLaneHaps) {
                tmpl.emplace_back();
                t = &tmpl.back();
                ln = 0;
              }
              t->lanes[ln].push_back(h);
              t->rows[ln] += n;
            }
          }
        }
        if (M.tmpl_geom >= 0) {
          const std::vector<LaneTemplate>& tmpl = M.tmpls[(M.tmpl_geom & kStripedBin) ? kMaxTilings - 1 : M.tmpl_geom];
          const int key = mode * kMaxTilings + ((M.tmpl_geom & kStripedBin) ? kMaxTilings - 1 : M.tmpl_geom);
          if (sbin_index[key] < 0) {
            sbin_index[key] = (int)ctx->sbins.size();
            ctx->sbins.push_back(phmm_ctx::SBin{mode, M.tmpl_geom, 0, 0});
          }
          const uint8_t sbi = (uint8_t)sbin_index[key];
          if (mode == kFast32) {                       // tilings its device-built units can use
            const int g64 = r64_geom_for(m), gx = rx32_geom_for(m);
            long64 |= m + 1 > kR64MaxW;
            long32 |= m + 1 > kRX32MaxW;
            if (g64 >= 0) { ctx->r64_geoms |= 1u << g64; r64_pairs[g64] += nh; }
            if (gx >= 0) { ctx->rx32_geoms |= 1u << gx; rx32_pairs[gx] += nh; }
          }
          for (const LaneTemplate& t : tmpl) {
            StreamUnit su;
            su.read = (int)r;
            su.list = (int)ctx->shaps.size();
            su.cntA = (int)t.lanes[0].size(); su.cntB = (int)t.lanes[1].size();
            su.rowsA = t.rows[0]; su.rowsB = t.rows[1];
            su.ro = (int)roff[r];
            su.m = m;
            for (int ln = 0; ln < 2; ++ln)
              for (int h : t.lanes[ln])
                ctx->shaps.push_back(StreamHap{h, (int)(gid + (h - h0)), (int)hoff[h], (int)ctx->hap_len[h]});
            ctx->su_all.push_back(su);
            ctx->su_bin.push_back(sbi);
          }
          continue;
        }
      }
      if (exact) {                                     // per-pair bit-exact kernels
        for (int64_t h = h0; h < h1; ++h) {
          ExactItem it{(int)(gid + (h - h0)), (int)r, (int)h, scale};
          (f64 ? host64 : host32)[exact_slot_host(m)].push_back(it);
        }
        continue;
      }
      for (int64_t x = 0; x < nh; x += 2) {
        const int ha = hidx[x], hb = (x + 1 < nh) ? hidx[x + 1] : hidx[x];
        FastUnit u;
        u.read = (int)r; u.hapA = ha; u.hapB = hb;
        u.pairA = (int)(gid + (ha - h0));
        u.pairB = (x + 1 < nh) ? (int)(gid + (hb - h0)) : -1;
        u.nA = (int)ctx->hap_len[ha]; u.nB = (int)ctx->hap_len[hb];
        u.pad = 0;
        int Q;
        const int g = choose_geom(m, std::max(u.nA, u.nB), &Q);
        const int key = g * 64 + std::min(Q, 63);
        if (bin_index[key] < 0) {
          bin_index[key] = (int)ctx->bins.size();
          ctx->bins.push_back(Bin{g, Q, {}, 0});
        }
        ctx->bins[bin_index[key]].units.push_back(u);
      }
    }
  }
  ctx->max_n = max_n;
  // LPT: costliest units first inside every bin; stable for determinism
  int64_t nunits = 0;
  for (auto& bn : ctx->bins) {
    std::stable_sort(bn.units.begin(), bn.units.end(), [](const FastUnit& a, const FastUnit& c) {
      return std::max(a.nA, a.nB) > std::max(c.nA, c.nB);
    });
    bn.dev_off = nunits;
    nunits += (int64_t)bn.units.size();
  }
  // LPT order per tiling: one stable counting sort on (bin, descending lane rows)
  const int nsbins = (int)ctx->sbins.size();
  const int64_t nsunits = (int64_t)ctx->su_all.size();
  std::vector<int> bmax(nsbins, 0), bbase(nsbins + 1, 0);
  for (int64_t i = 0; i < nsunits; ++i) {
    const StreamUnit& u = ctx->su_all[i];
    bmax[ctx->su_bin[i]] = std::max(bmax[ctx->su_bin[i]], std::max(u.rowsA, u.rowsB));
  }
  for (int bi = 0; bi < nsbins; ++bi) bbase[bi + 1] = bbase[bi] + bmax[bi] + 1;
  auto key = [&](int64_t i) {
    const StreamUnit& u = ctx->su_all[i];
    const int bi = ctx->su_bin[i];
    return bbase[bi] + bmax[bi] - std::max(u.rowsA, u.rowsB);
  };
  ctx->su_cnt.assign(bbase[nsbins] + 1, 0);
  for (int64_t i = 0; i < nsunits; ++i) ++ctx->su_cnt[key(i) + 1];
  for (int k = 1; k <= bbase[nsbins]; ++k) ctx->su_cnt[k] += ctx->su_cnt[k - 1];
  for (int bi = 0; bi < nsbins; ++bi) ctx->sbins[bi].dev_off = ctx->su_cnt[bbase[bi]];
  for (int bi = 0; bi < nsbins; ++bi)
    ctx->sbins[bi].count = (bi + 1 < nsbins ? ctx->su_cnt[bbase[bi + 1]] : nsunits) - ctx->sbins[bi].dev_off;
  ctx->h_sunits.resize(nsunits);
  for (int64_t i = 0; i < nsunits; ++i) ctx->h_sunits[ctx->su_cnt[key(i)]++] = ctx->su_all[i];
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
  std::vector<FastUnit> allu;
  allu.reserve(nunits);
  for (auto& bn : ctx->bins) allu.insert(allu.end(), bn.units.begin(), bn.units.end());
  CK(up(ctx->d_units, allu.data(), allu.size()));
  CK(up(ctx->d_sunits, ctx->h_sunits.data(), ctx->h_sunits.size()));
  CK(up(ctx->d_shaps, ctx->shaps.data(), ctx->shaps.size()));
  CK(ctx->d_gsum.ensure(R));
  CK(ctx->d_rflags.ensure(R));
  CK(ctx->d_acc.ensure(N));
  CK(ctx->d_status.ensure(N));
  CK(ctx->d_counters.ensure(kBinCounters + ctx->bins.size() + ctx->sbins.size()));
  for (int s = 0; s < kNumExactP; ++s) {
    ctx->list_cap[s] = (int)std::max<int64_t>(slot_pairs[s], 1);
    ctx->host_ex32[s] = (int)host32[s].size();
    ctx->host_ex64[s] = (int)host64[s].size();
    CK(ctx->d_ex32[s].ensure(ctx->list_cap[s]));
    CK(ctx->d_ex64[s].ensure(ctx->list_cap[s]));
    CK(ctx->d_fx64[s].ensure(ctx->list_cap[s]));
    if (!host32[s].empty()) CK(up(ctx->d_ex32[s], host32[s].data(), host32[s].size()));
    if (!host64[s].empty()) CK(up(ctx->d_ex64[s], host64[s].data(), host64[s].size()));
  }
  // boundary-column scratch: 2 buffers x 3 values x (max_n + 1) rows per sub-warp slot
  const int slots_per_sm = 4 * (kThreads / 32) * 8;   // <= 4 CTAs/SM x 4 warps x 8 sub-warps
  const size_t col_elems = (size_t)ctx->num_sms * slots_per_sm * 2 * 3 * (size_t)(max_n + 1);
  bool need_col = false, need_cold = false;
  for (auto& bn : ctx->bins) need_col |= bn.Q > 1;
  for (int s = 0; s < kNumExactP; ++s) need_cold |= true;
  if (need_col) CK(ctx->d_colf.ensure(col_elems));
  CK(ctx->d_cold.ensure(col_elems));   // exact kernels (f32 view uses half of it)
  (void)need_cold;
  trace.mark("plan-upload");
  // content validation on the device (bases 0..4, qualities 0..93)
  CK(ctx->d_vflag.ensure(1));
  int* vflag = ctx->d_vflag.p;                 // also gates every kernel of the execute
  CK(cudaMemsetAsync(vflag, 0, sizeof(int), ctx->stream));
  if (RL + HL > 0) {
    const int64_t work = std::max<int64_t>(RL, HL) / 16 + 1;
    const int vblocks = (int)std::min<int64_t>(ctx->num_sms * 8, (work + 255) / 256);
    k_validate<<<vblocks, 256, 0, ctx->stream>>>((const uint8_t*)ctx->d_rbases.p, ctx->d_bq.p, ctx->d_iq.p,
                                                 ctx->d_dq.p, ctx->d_gq.p, RL, (const uint8_t*)ctx->d_hbases.p,
                                                 HL, vflag);
    CK(cudaGetLastError());
  }
  CK(cudaMemcpyAsync(ctx->h_vflag, vflag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaEventRecord(ctx->ev_end, ctx->stream));
  ctx->h2d_bytes = bytes;
  ctx->h2d_ms = 0.0;
  if (!ctx->async) {
    int rc = check_validation(ctx);
    if (rc != PHMM_SUCCESS) return rc;
    float h2d = 0.f;
    cudaEventElapsedTime(&h2d, ctx->ev_start, ctx->ev_end);
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
  for (int g = 0; g < kNumR64Geoms; ++g)
    if (ctx->r64_geoms & (1u << g))   // widest tiling, long reads: a second region (r64b)
      CK(ctx->d_r64u[g].ensure(r64_pairs[g] * (g == kNumR64Geoms - 1 && long64 && rx32 ? 2 : 1)));
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
  E.band_budget = 2 * ctx->num_sms / std::max(1, ctx->budget_div);
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
    const bool big = streamed >= kBigCallPairs;
    L.lane_haps = &L == &E.r64 ? (big ? 4 : kRetryLaneHaps64) : (big ? 3 : kRetryLaneHapsX32);
  };
  lists(E.r64, ctx->d_r64u, kNumR64Geoms, ctx->d_r64h, ctx->r64_geoms, kCtrR64, r64_pairs);
  lists(E.rx32, ctx->d_rx32u, kNumRX32Geoms, ctx->d_rx32h, ctx->rx32_geoms, kCtrRX32, rx32_pairs);
  // second stage for long reads: guard-band pairs whose striped exact rerun underflows get
  // striped FP64 units in the upper half of the widest FP64 list (haplotype entries share
  // the first stage's array), run after the post-pass instead of the per-pair kernel
  {
    const int g = kNumR64Geoms - 1;
    E.r64b = E.r64;
    for (int x = 0; x < 8; ++x) E.r64b.units[x] = nullptr;
    E.r64b.count = ctx->d_counters.p + kCtrR64b;
    E.r64b.lane_haps = 1;
    E.r64b.enabled = (r64 && rx32 && long64 && (ctx->r64_geoms & (1u << g))) ? 1 : 0;
    if (E.r64b.enabled) E.r64b.units[g] = ctx->d_r64u[g].p + r64_pairs[g];
  }
  // grids of the stream launches, and boundary-column space for the ones that can meet
  // striped units (reads longer than the tiling width): per sub-warp slot 2 columns x
  // 3 states x (row capacity + 1) two-lane values
  {
    int64_t col_total = 0;
    auto col_bytes = [&](int mode, const StreamKernel& K, int grid) -> int64_t {
      const int64_t v = (mode == kFast64 || mode == kExact64) ? 16 : 8;
      return (int64_t)grid * 4 * (32 / K.P) * 6 * col_rows_for(K.P) * v;
    };
    for (auto& sb : ctx->sbins) {
      const StreamKernel& K = skern(sb.mode, sb.geom);
      const int G = 32 / K.P;
      const int64_t groups = (sb.count + G - 1) / G;
      const bool striped = (sb.geom & kStripedBin) != 0;
      // striped bins with few units run in team mode (a CTA per unit): one CTA per unit
      const int64_t want = striped && groups * 2 <= (int64_t)ctx->num_sms * K.occ * 4 ? groups : (groups + 3) / 4;
      sb.grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->num_sms * K.occ, want));
      sb.col_off = striped ? col_total : -1;
      if (striped) col_total += col_bytes(sb.mode, K, sb.grid);
    }
    for (int g = 0; g < 8; ++g) { ctx->r64_col_off[g] = -1; ctx->rx32_col_off[g] = -1; }
    if (long64) {                                   // reads > 255 stripe on the widest FP64 tiling
      const int g = kNumR64Geoms - 1;
      if (ctx->r64_geoms & (1u << g)) {
        ctx->r64_col_off[g] = col_total;
        col_total += col_bytes(kFast64, kStripedTab[kFast64], ctx->num_sms * kStripedTab[kFast64].occ);
      }
    }
    if (long32) {                                   // reads > 511: exact FP32 stripes
      const int g = kNumRX32Geoms - 1;
      if (ctx->rx32_geoms & (1u << g)) {
        ctx->rx32_col_off[g] = col_total;
        col_total += col_bytes(kExact32, kStripedTab[kExact32], ctx->num_sms * kStripedTab[kExact32].occ);
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

int phmm_execute(phmm_ctx* ctx) {
  if (!ctx) return PHMM_ERR_INVALID;
  if (!ctx->prepared) return ctx->fail(PHMM_ERR_STATE, "phmm_execute before phmm_prepare");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const EngineDev& E = ctx->dev;
  const int64_t N = ctx->num_pairs;
  int launches = 0;
  // counters: [0,4) ex32 counts, [4,8) ex64 counts, [8,12) ex32 work, [12,16) ex64 work,
  // 16 inline guard-band pairs, [20,24) fx64 counts, [24,28) fx64 work, [32,38) FP64
  // stream-retry unit counts, 38 their haplotype count, [40,46) their work counters,
  // [kBinCounters, +bins) fast-kernel bins
  const int nb = (int)ctx->bins.size();
  std::vector<int> blocks(nb, 0);
  for (int bi = 0; bi < nb; ++bi) {
    const Bin& bn = ctx->bins[bi];
    const int nu = (int)bn.units.size();
    if (nu == 0) continue;
    const int G = 32 / kFastGeoms[bn.geom].P;
    const int groups = (nu + G - 1) / G;
    blocks[bi] = std::max(1, std::min(ctx->num_sms * kFastOcc[bn.geom], (groups + 3) / 4));
  }
  CK(cudaEventRecord(ctx->ev_start, st));
  const int nsb = (int)ctx->sbins.size();
  int* bin_ctr = ctx->d_counters.p + kBinCounters;
  // counters (host list sizes in [0, 8), zero elsewhere) and per-pair status are reset by
  // k_precompute itself: no small H2D copy / memsets on the critical path
  const int4 hc0 = make_int4(ctx->host_ex32[0], ctx->host_ex32[1], ctx->host_ex32[2], ctx->host_ex32[3]);
  const int4 hc1 = make_int4(ctx->host_ex64[0], ctx->host_ex64[1], ctx->host_ex64[2], ctx->host_ex64[3]);
  // L2 prefetch of the per-unit inputs on a side stream, beside k_precompute (joined with
  // the FP32 phase; the bench flushes L2 between steps)
  CK(cudaEventRecord(ctx->ev_pre, st));
  CK(cudaStreamWaitEvent(ctx->aux[phmm_ctx::kAux - 1], ctx->ev_pre, 0));
  k_l2_prefetch<<<ctx->num_sms * 2, 256, 0, ctx->aux[phmm_ctx::kAux - 1]>>>(
      ctx->d_sunits.p, (int64_t)ctx->h_sunits.size() * (int64_t)sizeof(StreamUnit), ctx->d_shaps.p,
      (int64_t)ctx->shaps.size() * (int64_t)sizeof(StreamHap), ctx->d_hbases.p, ctx->hap_bytes, ctx->d_rbases.p,
      ctx->d_bq.p, ctx->read_bytes);
  ++launches;
  {
    const int threads = 128;
    const int64_t blocks_pre = std::max<int64_t>(1, (ctx->num_reads * 32 + threads - 1) / threads);
    k_precompute<<<(unsigned)blocks_pre, threads, 0, st>>>(E, (int)ctx->num_reads, ctx->d_counters.p,
                                                           kBinCounters + nb + nsb, hc0, hc1, N);
    ++launches;
  }
  CK(cudaEventRecord(ctx->ev_pre, st));
  CK(cudaEventRecord(ctx->ev_fast0, st));
  // Fast-kernel bins (one persistent launch per tiling) go round-robin onto side streams
  // so a bin's tail (its last CTAs draining) overlaps the next bin's work.  Legacy k_fast
  // bins share the boundary-column scratch: they stay serialized on the last side stream.
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
               bin_ctr + nb + bi, sb.col_off >= 0 ? ctx->d_colstream.p + sb.col_off : nullptr,
               col_rows_for(SKn.P));
    ++launches;
  }
  for (int bi = 0; bi < nb; ++bi) {
    const Bin& bn = ctx->bins[bi];
    const int nu = (int)bn.units.size();
    if (nu == 0) continue;
    used[phmm_ctx::kAux - 1] = true;
    kFastLaunch[bn.geom](dim3(blocks[bi]), fast_smem(bn.geom), ctx->aux[phmm_ctx::kAux - 1], E,
                         ctx->d_units.p + bn.dev_off, nu, bn.Q, bin_ctr + bi, ctx->d_colf.p, ctx->max_n + 1);
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
  k_exact_all<float><<<ctx->num_sms * 2, kThreads, exact_smem(0, 4), ctx->aux[0]>>>(
      E, ctx->d_counters.p + 8, (float*)ctx->d_cold.p, ctx->max_n + 1);
  ++launches;
  int nside = 0;
  auto post = [&](const StreamKernel& SKn, const RetryLists& L, int g, int* work, int64_t col_off) {
    const int a = 1 + (nside++ % (phmm_ctx::kAux - 1));
    used[a] = true;
    SKn.launch(dim3(ctx->num_sms * SKn.occ), SKn.smem, ctx->aux[a], E, L.units[g], L.haps, L.unit_cap[g], L.count + g,
               work, col_off >= 0 ? ctx->d_colstream.p + col_off : nullptr, col_rows_for(SKn.P));
    ++launches;
  };
  for (int g = kNumR64Geoms - 1; g >= 0; --g)
    if (ctx->r64_geoms & (1u << g))
      post(ctx->r64_col_off[g] >= 0 ? kStripedTab[kFast64] : kStreamFast64[g], E.r64, g,
           ctx->d_counters.p + kCtrR64Work + g, ctx->r64_col_off[g]);
  for (int g = kNumRX32Geoms - 1; g >= 0; --g)
    if (ctx->rx32_geoms & (1u << g))
      post(ctx->rx32_col_off[g] >= 0 ? kStripedTab[kExact32] : kStreamExact32[g], E.rx32, g,
           ctx->d_counters.p + kCtrRX32Work + g, ctx->rx32_col_off[g]);
  CK(join());
  if (E.r64b.enabled) {                 // long reads: band pairs whose exact rerun underflowed
    const int g = kNumR64Geoms - 1;
    const StreamKernel& SKn = kStripedTab[kFast64];
    SKn.launch(dim3(ctx->num_sms * SKn.occ), SKn.smem, st, E, E.r64b.units[g], E.r64b.haps, E.r64b.unit_cap[g],
               E.r64b.count + g, ctx->d_counters.p + kCtrR64bWork + g, ctx->d_colstream.p + ctx->r64_col_off[g],
               col_rows_for(SKn.P));
    ++launches;
  }
  if (ctx->flags & PHMM_FLAG_RETRY_F64) {
    k_fast64_all<<<ctx->num_sms * 2, kThreads, exact_smem(0, 8), st>>>(E, ctx->d_counters.p + 24, ctx->d_cold.p,
                                                                      ctx->max_n + 1);
    ++launches;
  }
  k_exact_all<double><<<ctx->num_sms * 2, kThreads, exact_smem(0, 8), st>>>(
      E, ctx->d_counters.p + 12, ctx->d_cold.p, ctx->max_n + 1);
  ++launches;
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev_end, st));
  ctx->last_launches = launches;
  ctx->executed = true;
  if (ctx->async) return PHMM_SUCCESS;
  CK(cudaEventSynchronize(ctx->ev_end));
  float dev = 0.f, fast = 0.f;
  CK(cudaEventElapsedTime(&dev, ctx->ev_start, ctx->ev_end));
  CK(cudaEventElapsedTime(&fast, ctx->ev_fast0, ctx->ev_fast1));
  ctx->last_dev_ms = dev;
  ctx->last_fast_ms = fast;
  return PHMM_SUCCESS;
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
  CK(cudaEventRecord(ctx->ev_fast0, ctx->stream));     // (reused as the D2H start marker)
  if (N > 0) {
    CK(cudaMemcpyAsync(ctx->h_acc, ctx->d_acc.p, N * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(ctx->h_st, ctx->d_status.p, N, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaEventRecord(ctx->ev_fast1, ctx->stream));
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
  CK(cudaEventSynchronize(ctx->ev_fast1));
  float d2h = 0.f;
  cudaEventElapsedTime(&d2h, ctx->ev_fast0, ctx->ev_fast1);
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
    for (auto& bn : ctx->bins) {
      const FastGeom g = kFastGeoms[bn.geom];
      for (auto& u : bn.units) comp += 2LL * bn.Q * g.P * g.K * (std::max(u.nA, u.nB) + g.P - 1);
    }
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

int phmm_fast_geometry(int m, int n, int* P, int* K, int* Q) {
  if (m < 1 || n < 1 || !P || !K || !Q) return PHMM_ERR_INVALID;
  int q = 1;
  const int g = choose_geom(m, n, &q);
  *P = kFastGeoms[g].P; *K = kFastGeoms[g].K; *Q = q;
  return PHMM_SUCCESS;
}

// phmm_score pipelines large calls: the batches are cut into kScoreChunks contiguous
// chunks of ~equal pair count, each scored by its own chunk context (device buffers,
// streams, pinned staging).  The host plans chunk c+1 while the GPU uploads and scores
// chunk c, and finishes chunk c while later chunks run; chunk kernels on separate
// streams also fill each other's tails.  Results are identical to the one-pass path
// (pairs are independent; gid order is batch-major, so a chunk owns a gid range).
static int score_chunked(phmm_ctx* ctx, const phmm_input* in, const phmm_options* opt, double* out_log10,
                         uint8_t* out_status, phmm_stats* stats, int nchunks) {
  const int64_t B = in->num_batches;
  std::vector<int64_t> pairs(B + 1, 0);
  for (int64_t b = 0; b < B; ++b)
    pairs[b + 1] = pairs[b] + (in->batch_read_off[b + 1] - in->batch_read_off[b]) *
                                  (in->batch_hap_off[b + 1] - in->batch_hap_off[b]);
  const int64_t N = pairs[B];
  std::vector<int64_t> cut(nchunks + 1, B);
  cut[0] = 0;
  for (int c = 1; c < nchunks; ++c) {
    int64_t b = cut[c - 1];
    while (b < B && pairs[b] < N * c / nchunks) ++b;
    cut[c] = std::max(b, cut[c - 1]);
  }
  while ((int)ctx->chunks.size() < nchunks) {
    phmm_ctx* c = new (std::nothrow) phmm_ctx();
    if (!c) return ctx->fail(PHMM_ERR_NOMEM, "chunk context");
    c->lut = ctx->lut;
    c->parent = ctx;
    ctx->chunks.push_back(c);
    const int rc = init_ctx(c, ctx->device);
    if (rc != PHMM_SUCCESS) return ctx->fail(rc, "chunk context: %s", c->err.c_str());
    c->async = true;
  }
  // enqueue every chunk (prepare + execute + D2H), planning the next one meanwhile
  for (int c = 0; c < nchunks; ++c) {
    phmm_ctx* cx = ctx->chunks[c];
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
    cx->budget_div = nchunks;
    int rc = phmm_prepare(cx, &sub, opt, &n);
    if (rc == PHMM_SUCCESS) rc = phmm_execute(cx);
    if (rc == PHMM_SUCCESS) rc = fetch_enqueue(cx);
    if (rc != PHMM_SUCCESS) return ctx->fail(rc, "%s", cx->err.c_str());
  }
  // complete in order: device validation verdict, then finishing into the caller's slice
  phmm_stats total;
  memset(&total, 0, sizeof(total));
  for (int c = 0; c < nchunks; ++c) {
    phmm_ctx* cx = ctx->chunks[c];
    if (cut[c + 1] <= cut[c]) continue;
    int rc = check_validation(cx);
    if (rc != PHMM_SUCCESS) return ctx->fail(rc, "%s", cx->err.c_str());
    phmm_stats cs;
    const int64_t g0 = pairs[cut[c]];
    rc = fetch_complete(cx, out_log10 ? out_log10 + g0 : nullptr, out_status ? out_status + g0 : nullptr, &cs);
    if (rc != PHMM_SUCCESS) return ctx->fail(rc, "%s", cx->err.c_str());
    total.num_pairs += cs.num_pairs; total.total_cells += cs.total_cells;
    total.computed_cells += cs.computed_cells; total.fast_pairs += cs.fast_pairs;
    total.exact_pairs += cs.exact_pairs; total.f64_pairs += cs.f64_pairs;
    total.flagged_pairs += cs.flagged_pairs; total.h2d_bytes += cs.h2d_bytes; total.d2h_bytes += cs.d2h_bytes;
    total.kernel_launches += cs.kernel_launches; total.plan_ms += cs.plan_ms; total.d2h_ms += cs.d2h_ms;
  }
  if (stats) *stats = total;
  return PHMM_SUCCESS;
}

int phmm_score(phmm_ctx* ctx, const phmm_input* in, const phmm_options* opt, double* out_log10,
               uint8_t* out_status, phmm_stats* stats) {
  if (!ctx) return PHMM_ERR_INVALID;
  if (in && opt && in->num_batches >= 2 * std::max(3, score_chunks()) && score_chunks() != 1 && in->batch_read_off && in->batch_hap_off &&
      in->read_off && in->hap_off && score_chunking_enabled()) {
    // validate the structure first (the chunk views index the offset arrays)
    int64_t pairs = 0;
    bool ok = in->batch_read_off[0] == 0 && in->batch_hap_off[0] == 0 &&
              in->batch_read_off[in->num_batches] == in->num_reads &&
              in->batch_hap_off[in->num_batches] == in->num_haps && in->read_off[0] == 0 && in->hap_off[0] == 0;
    for (int64_t b = 0; ok && b < in->num_batches; ++b) {
      const int64_t nr = in->batch_read_off[b + 1] - in->batch_read_off[b];
      const int64_t nh = in->batch_hap_off[b + 1] - in->batch_hap_off[b];
      ok = nr > 0 && nh > 0;
      pairs += nr * nh;
    }
    // Only regular calls are pipelined: reads spanning many tiling widths split into many
    // small per-tiling kernels per chunk, and each chunk's latency-bound post-pass (guard
    // band, FP64 retries) then queues behind the next chunks' persistent grids.
    if (ok && pairs >= kScoreChunkMinPairs) {
      static const int kW[] = {16, 32, 48, 64, 80, 96, 112, 128, 160, 192, 224, 256, 320, 384, 448, 512};
      unsigned classes = 0;
      for (int64_t r = 0; r < in->num_reads; ++r) {
        const int64_t m = in->read_off[r + 1] - in->read_off[r];
        int c = 0;
        while (c < 15 && kW[c] < m + 1) ++c;
        classes |= 1u << c;
      }
      // large calls amortize the per-chunk post-pass latency: pipeline them regardless
      ok = __builtin_popcount(classes) <= 2 || pairs >= kBigCallPairs;
    }
    if (ok && pairs >= kScoreChunkMinPairs) {
      CK(cudaSetDevice(ctx->device));
      // per-chunk planning overhead vs pipeline depth: 3 chunks for ordinary calls, 4 for
      // large ones (c2: 3 -> +15 % e2e over 4; c5: 4 -> +6 % over 3)
      const int nch = score_chunks() > 0 ? score_chunks() : (pairs >= kBigCallPairs ? 4 : 3);
      return score_chunked(ctx, in, opt, out_log10, out_status, stats, nch);
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
