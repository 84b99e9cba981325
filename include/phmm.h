/*
 * phmm.h — C-ABI of the B200 Pair-HMM forward engine (libphmm.so).
 *
 * The reference (arxiv 2411.11547 artifact, /root/reference/pkg) has no native
 * FFI: its hot path is Python -> numba.  These entry points replace, as one
 * native call, the engine half of its batch-likelihood API:
 *
 *   phmm_score   replaces  pipeline.run's work loop            pipeline.py:90-142
 *                           (enumerate_work_items               model.py:123-136,
 *                            _assign / select_config             partition.py:20-37,62-85,
 *                            forward_wavefront_batch             wavefront.py:453-505,
 *                            stage_read / build_transitions /    wavefront.py:332-365,
 *                            build_emission_table                prob.py:66-112,
 *                            _kernel                             wavefront.py:61-315,
 *                            _finish_value + scatter             wavefront.py:428-434,474-479)
 *   phmm_prepare / phmm_execute / phmm_fetch
 *                split phmm_score into upload+plan, device-resident compute and
 *                download, so callers can time the kernels with inputs already in HBM.
 *   phmm_create / phmm_destroy / phmm_last_error   context plumbing (device, streams,
 *                device buffers, the Phred LUT of prob.py:36).
 *
 * Conventions: plain pointers and sizes; the caller owns every host buffer; the
 * library owns device memory inside the opaque context.  Every call returns a
 * PHMM_* return code; phmm_last_error() gives the message.  A context is
 * single-caller (not thread-safe) and bound to one CUDA device.
 *
 * Per-pair results follow the reference's run() semantics: out_log10[gid] is
 * log10(acc) - scale_log2*log10(2) (wavefront.py:428-434), NaN for failed pairs,
 * and out_status[gid] holds the error kind (errors.py:8-61) in its low nibble.
 */
#ifndef PHMM_H_
#define PHMM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PHMM_ABI_VERSION 1

/* return codes */
#define PHMM_SUCCESS 0
#define PHMM_ERR_INVALID (-1)   /* malformed input or options (errors.py "data") */
#define PHMM_ERR_CUDA (-2)      /* CUDA runtime failure / no device */
#define PHMM_ERR_NOMEM (-3)     /* device or host allocation failed */
#define PHMM_ERR_STATE (-4)     /* call order (execute before prepare, ...) */

/* per-pair status, low nibble = error kind (errors.py), high bits = provenance */
#define PHMM_ST_OK 0
#define PHMM_ST_NUMERIC_OVERFLOW 1      /* errors.py:54-57 "numeric-overflow" */
#define PHMM_ST_CONFIG_TOO_SMALL 2      /* errors.py:38-41 "config-too-small" */
#define PHMM_ST_DEGENERATE 3            /* errors.py:32-35 "degenerate-transition" */
#define PHMM_ST_KIND_MASK 0x0F
#define PHMM_ST_EXACT_F32 0x20          /* value from the bit-exact FP32 kernel (guard band) */
#define PHMM_ST_RETRIED_F64 0x40        /* FP32 underflowed; value from the FP64 retry pass */

/* option flags */
#define PHMM_FLAG_RETRY_F64 0x1   /* rerun FP32-underflowing pairs in FP64 (GATK behaviour) */
#define PHMM_FLAG_EXACT 0x2       /* every FP32 pair on the bit-exact kernel (no fast path) */

typedef struct phmm_ctx phmm_ctx;

/* Flat batch list.  Reads r occupy [read_off[r], read_off[r+1]) of the base and
 * quality arrays; haplotypes likewise; batch b owns reads
 * [batch_read_off[b], batch_read_off[b+1]) and haps [batch_hap_off[b], ...).
 * Pair global ids enumerate batch-major, read-major, hap-minor (model.py:123-136). */
typedef struct {
  const int8_t* read_bases;   /* codes A=0 C=1 G=2 T=3 N=4 (model.py:14-18) */
  const uint8_t* base_qual;   /* Phred 0..93 */
  const uint8_t* ins_qual;
  const uint8_t* del_qual;
  const uint8_t* gcp_qual;
  const int64_t* read_off;    /* num_reads + 1 */
  int64_t num_reads;
  const int8_t* hap_bases;
  const int64_t* hap_off;     /* num_haps + 1 */
  int64_t num_haps;
  const int64_t* batch_read_off; /* num_batches + 1 */
  const int64_t* batch_hap_off;  /* num_batches + 1 */
  int64_t num_batches;
} phmm_input;

/* Registered configurations (model.py:139-193).  Each read binds to the smallest
 * p*k >= m, ties to fewer lanes (partition.py:20-37); the bound config supplies
 * the read's precision (0 = f32, 1 = f64) and boundary scale 2^scale_log2.
 * The engine's own tiling is independent of (p, k): scores are tiling-invariant
 * (test_acceptance.py:88-103). */
typedef struct {
  int32_t num_configs;
  const int32_t* p;
  const int32_t* k;
  const int32_t* precision;
  const int32_t* scale_log2;
  int32_t flags;              /* PHMM_FLAG_* */
} phmm_options;

typedef struct {
  int64_t num_pairs;
  int64_t total_cells;        /* true m*n over executed pairs (pipeline.py:103-111) */
  int64_t computed_cells;     /* cells the kernels evaluated, padding included */
  int64_t fast_pairs;         /* accepted from the FP32 fast kernel */
  int64_t exact_pairs;        /* evaluated by the bit-exact FP32 kernel */
  int64_t f64_pairs;          /* evaluated in FP64 (f64 configs + retries) */
  int64_t flagged_pairs;      /* FP32 numeric-overflow (before any retry) */
  int64_t h2d_bytes;
  int64_t d2h_bytes;
  int32_t kernel_launches;    /* engine kernels launched by the last execute */
  int32_t reserved;
  double device_ms;           /* last execute: CUDA-event time of the kernel work */
  double fast_ms;             /* of which the FP32 fast kernels */
  double h2d_ms, d2h_ms, plan_ms;
} phmm_stats;

int phmm_abi_version(void);

/* phred_lut: 94 doubles, PHRED_TO_PROB of prob.py:36 (pass the caller's table so
 * the engine uses bit-identical probabilities). */
int phmm_create(phmm_ctx** ctx, int device, const double* phred_lut);
int phmm_destroy(phmm_ctx* ctx);
const char* phmm_last_error(const phmm_ctx* ctx);

/* One call = prepare + execute + fetch. out_log10 / out_status: num_pairs entries. */
int phmm_score(phmm_ctx* ctx, const phmm_input* in, const phmm_options* opt,
               double* out_log10, uint8_t* out_status, phmm_stats* stats);

/* Bound the device working set of phmm_score (bytes; 0 = no bound, the default).  A call
 * whose estimated footprint exceeds the bound streams through at most three chunk
 * contexts reused round-robin, each chunk within a third of the bound (a single batch
 * larger than that is one chunk); without a bound the same happens automatically when a
 * call would not fit the free device memory.  Replaces the reference's chunk budget
 * (partition.py:88-119, pipeline.py:116-136: contiguous global-id chunks, each within the
 * budget, the next staged while the current one computes) for inputs larger than HBM. */
int phmm_set_device_budget(phmm_ctx* ctx, int64_t bytes);
/* Pipelining depth of phmm_score: 0 (the default) = automatic -- calls of >= 2^20 pairs
 * stream through six chunk contexts with ramped sizes (1,3,5,5,3,1)/18, so host planning,
 * H2D, kernels and the host finishing of different chunks overlap; smaller calls run one
 * pass.  n in 2..8 pipelines every call of >= 2n batches through n equal chunks (results
 * are identical either way: pairs are independent).  1 = never pipeline. */
int phmm_set_pipeline(phmm_ctx* ctx, int n);
/* Page-lock (pin) / release a caller-owned host buffer so the uploads from it are DMA
 * transfers that overlap the host planning (cudaHostRegister).  For buffers a caller
 * reuses across calls (the Python run() flattening arena); pinned-allocated buffers need
 * neither. */
int phmm_pin_host(void* ptr, int64_t bytes);
int phmm_unpin_host(void* ptr);
/* Device bytes currently allocated by the context and its chunk contexts. */
int phmm_device_bytes(const phmm_ctx* ctx, int64_t* bytes);

/* Upload inputs and build the work plan; returns the pair count in *num_pairs. */
int phmm_prepare(phmm_ctx* ctx, const phmm_input* in, const phmm_options* opt,
                 int64_t* num_pairs);
/* Run every kernel of the prepared plan on device-resident data (re-runnable). */
int phmm_execute(phmm_ctx* ctx);
/* CUDA-event timings of the last phmm_execute (engine stream): whole execute, the
 * FP32 fast kernels alone, and the number of engine kernels launched. */
int phmm_last_timing(const phmm_ctx* ctx, double* device_ms, double* fast_ms, int* launches);
/* Per-phase CUDA-event timings of the last phmm_execute (engine stream), 4 doubles (ms):
 * [0] k_precompute (+ L2 prefetch), [1] FP32 stream phase (all tiling bins, concurrent),
 * [2] post-pass (a): device-built exact-FP32 guard-band reruns and FP64 retry units,
 * concurrent, [3] post-pass (b)+(c): second-stage FP64 units, per-pair FP64 retries and
 * bit-exact FP64.  Replaces nothing in the reference (its RunReport.per_config holds
 * wall seconds per config, pipeline.py:116-124); measurement only. */
int phmm_last_phases(const phmm_ctx* ctx, double* phase_ms);
/* Download and finish the last execute's results. */
int phmm_fetch(phmm_ctx* ctx, double* out_log10, uint8_t* out_status, phmm_stats* stats);

/* The complete (m+1) x (n+1) FP64 dynamic-programming matrices M, I, D of ONE pair
 * (row-major, boundaries included), bit-identical to the reference's debugging oracle
 * forward_matrices (reference.py:150-156, _full_kernel reference.py:36-75) with boundary
 * 2^scale_log2 / n and the f64 flush (prob.py:39).  Caller-owned outputs of (m+1)*(n+1)
 * doubles each; the GPU kernel k_matrices computes them (debugging path, one CTA). */
int phmm_forward_matrices(phmm_ctx* ctx, const int8_t* read_bases, const uint8_t* base_qual,
                          const uint8_t* ins_qual, const uint8_t* del_qual, const uint8_t* gcp_qual, int32_t m,
                          const int8_t* hap_bases, int32_t n, int32_t scale_log2, double* M, double* I, double* D);

/* The fast kernel's tiling for a read of length m against haplotypes of length <= n:
 * P threads per sub-warp, K read positions per thread, Q stripes (no device needed).
 * Replaces the reference's per-config step count (wavefront.py:314-315, steps = n + p):
 * the engine executes n + P - 1 wavefront steps per stripe. */
int phmm_fast_geometry(int m, int n, int* P, int* K, int* Q);

#ifdef __cplusplus
}
#endif

#endif /* PHMM_H_ */
