/*
 * ktune_b200.h -- the C-ABI drop-in boundary of the B200 build of ISAAC's
 * GEMM/CONV tuning path (paper_1802_05371_b200/libktune_b200.so).
 *
 * The reference (ktune, /root/reference/proj) is a C++20 library with no FFI
 * of its own; a C++ host that wants its GEMM/CONV path on the GPU crosses to
 * the device exactly where the reference calls its executors and its
 * measurement backend.  Every entry point below names the reference
 * interface it replaces (file:line under /root/reference/proj).  The C++
 * adapter a maintainer would add (a MeasurementBackend subclass and a
 * ctypes binding) is shown in INTEGRATION.md.
 *
 * Conventions
 *  - plain C types only; structs mirror the reference types field-for-field
 *    in canonical order (param_space.hpp:20-106);
 *  - every function returns a ktune_status; on failure ktune_last_error()
 *    returns a thread-local message (the reference's exception what());
 *  - "device" pointers are CUDA device pointers owned by the caller, and
 *    `stream` is a cudaStream_t (NULL = legacy default stream);
 *  - no CPU fallback: if the CUDA kernels cannot run, calls fail with
 *    KTUNE_ERR_CUDA.
 */
#ifndef KTUNE_B200_H
#define KTUNE_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define KTUNE_API __attribute__((visibility("default")))
#else
#define KTUNE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define KTUNE_B200_ABI_VERSION 1

/* Error classes of the reference, as codes (backends.cpp:120-125, 220-240,
 * 504-506; pipeline.cpp runtime_error paths). */
typedef enum ktune_status {
    KTUNE_OK = 0,
    KTUNE_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument: illegal tuning, size mismatch, bad field */
    KTUNE_ERR_UNSUPPORTED = 2,      /* dtype/tuple this build cannot execute ("cpu backend does not execute f16") */
    KTUNE_ERR_CUDA = 3,             /* a CUDA call failed */
    KTUNE_ERR_RUNTIME = 4,          /* std::runtime_error: malformed file, IO */
    KTUNE_ERR_WORKSPACE = 5         /* caller workspace smaller than *_workspace_size() */
} ktune_status;

/* Dtype of param_space.hpp:15 (f16/f32/f64) plus the tensor-core extensions. */
typedef enum ktune_dtype {
    KTUNE_F16 = 0,
    KTUNE_F32 = 1,
    KTUNE_F64 = 2,
    KTUNE_BF16 = 3,
    KTUNE_TF32 = 4
} ktune_dtype;

/* FAST: FFMA (SIMT) / tensor cores.  PARITY: bit-identical to the reference
 * executors execute_gemm<T>/execute_conv<T> (f32/f64 only). */
typedef enum ktune_mode { KTUNE_MODE_FAST = 0, KTUNE_MODE_PARITY = 1 } ktune_mode;

/* GemmInput, param_space.hpp:20-30. */
typedef struct ktune_gemm_input {
    int64_t m, n, k;
    int32_t dtype; /* ktune_dtype */
    int32_t trans_a;
    int32_t trans_b;
    int32_t reserved;
} ktune_gemm_input;

/* ConvInput, param_space.hpp:34-49 (valid mode: H = P+R-1, W = Q+S-1). */
typedef struct ktune_conv_input {
    int64_t n_batch, p, q, k_filters, c, r, s;
    int32_t dtype;
    int32_t reserved;
} ktune_conv_input;

/* GemmTuning, param_space.hpp:55-67 (canonical order m_s n_s m_l n_l u k_s k_l k_g). */
typedef struct ktune_gemm_tuning {
    int32_t m_s, n_s, m_l, n_l, u, k_s, k_l, k_g;
} ktune_gemm_tuning;

/* ConvTuning, param_space.hpp:69-77. */
typedef struct ktune_conv_tuning {
    int32_t k_s, p_s, q_s, n_s, k_l, p_l, q_l, n_l, u, c_s, c_l, c_g;
} ktune_conv_tuning;

/* HardwareDescriptor, param_space.hpp:87-106. */
typedef struct ktune_hw {
    int64_t max_shared_bytes_per_block;
    int64_t max_registers_per_thread;
    int64_t max_threads_per_block;
    int64_t max_warps_per_multiprocessor;
    int64_t warp_size;
    double alu_latency, alu_throughput, mem_latency, mem_throughput, clock_hz;
    int64_t num_multiprocessors;
} ktune_hw;

/* ResourceUsage, param_space.hpp:108-114. */
typedef struct ktune_resources {
    int64_t shared_bytes, registers_per_thread, threads_per_block;
} ktune_resources;

/* Options of a device measurement (CpuBackend ctor, backends.hpp:128-137,
 * plus the device-timing knobs the reference does not need). */
typedef struct ktune_measure_options {
    int32_t mode;        /* ktune_mode */
    int32_t repetitions; /* timed runs, best-of (reference default 3) */
    int32_t warmup;      /* untimed runs first (reference: 1) */
    int32_t flush_l2;    /* write-sweep L2 before each timed run */
    uint64_t seed;       /* operand fill seed (reference: 0x5eed) */
} ktune_measure_options;

/* ---- library ------------------------------------------------------------ */
KTUNE_API int ktune_abi_version(void);
KTUNE_API const char* ktune_last_error(void);
/* Selects the CUDA device used by subsequent host-buffer / measurement calls. */
KTUNE_API int ktune_set_device(int device);

/* ---- parameter space (param_space.cpp) ----------------------------------- */
/* HardwareDescriptor::from_json_text / defaults (param_space.cpp:140-178). */
KTUNE_API int ktune_hw_default(ktune_hw* out);
KTUNE_API int ktune_hw_from_json(const char* json_text, ktune_hw* out);
/* estimate_resources (param_space.cpp:204-231). */
KTUNE_API int ktune_estimate_resources_gemm(const ktune_gemm_input* in, const ktune_gemm_tuning* t, ktune_resources* out);
KTUNE_API int ktune_estimate_resources_conv(const ktune_conv_input* in, const ktune_conv_tuning* t, ktune_resources* out);
/* is_legal (param_space.cpp:275-314): *accepted 0/1, *reason = RejectReason
 * (0 divisibility, 1 shared_memory, 2 registers, 3 threads); detail text via
 * ktune_last_text(). */
KTUNE_API int ktune_is_legal_gemm(const ktune_hw* hw, const ktune_gemm_input* in, const ktune_gemm_tuning* t, int* accepted,
                        int* reason);
KTUNE_API int ktune_is_legal_conv(const ktune_hw* hw, const ktune_conv_input* in, const ktune_conv_tuning* t, int* accepted,
                        int* reason);
KTUNE_API const char* ktune_last_text(void);
/* enumerate_legal (param_space.cpp:536-628); bounds_json NULL/"" = defaults
 * (powers of two 1..16).  Writes min(count, cap) tunings; *count = total. */
KTUNE_API int ktune_enumerate_legal_gemm(const ktune_hw* hw, const ktune_gemm_input* in, const char* bounds_json,
                               ktune_gemm_tuning* out, int64_t cap, int64_t* count);
KTUNE_API int ktune_enumerate_legal_conv(const ktune_hw* hw, const ktune_conv_input* in, const char* bounds_json,
                               ktune_conv_tuning* out, int64_t cap, int64_t* count);
/* encode_features gemm.v1 (14) / conv.v1 (19) (param_space.cpp:630-659). */
KTUNE_API int ktune_encode_features_gemm(const ktune_gemm_input* in, const ktune_gemm_tuning* t, double* out14);
KTUNE_API int ktune_encode_features_conv(const ktune_conv_input* in, const ktune_conv_tuning* t, double* out19);
/* build_indirection_table (backends.cpp:197-216): 4 int64 per entry
 * {c, r, s, image_offset}; cap in entries, *count = C*R*S. */
KTUNE_API int ktune_build_indirection_table(const ktune_conv_input* in, int64_t* out4, int64_t cap, int64_t* count);

/* ---- device kernels (replace execute_gemm / execute_conv, backends.cpp:228-444) */
/* Workspace for k_g / c_g partials (0 bytes when the reduction is not split
 * across the grid): a 1 MiB region of per-tile arrival counters, then the
 * partials of every slice; the slice that arrives last folds them in slice
 * order and resets its counter (FAST with >= 16 slices instead adds the
 * partials into an accumulator in the upper half of the counter region with
 * L2 reductions; the last arrival stores C and re-zeroes it).  The counter
 * region (the first 1 MiB) must be zero before a workspace's first use --
 * allocate with cudaMemset 0 -- and every launch leaves it zero.  One launch
 * at a time per workspace. */
/* Launch geometry the library would use for this input/tuning (no launch):
 * threads per block, dynamic shared memory, grid {x, y, z}, and the kernel
 * family ("simt", "simt-tma", "simt-generic", "tcgen05", "tcgen05-pair"),
 * NUL-terminated into family[0..family_cap).  Reporting aid for tools. */
KTUNE_API int ktune_gemm_launch_info(const ktune_gemm_input* in, const ktune_gemm_tuning* t, int mode, int* threads,
                                     size_t* smem_bytes, int* grid3, char* family, size_t family_cap);
KTUNE_API int ktune_gemm_workspace_size(const ktune_gemm_input* in, const ktune_gemm_tuning* t, size_t* bytes);
KTUNE_API int ktune_conv_workspace_size(const ktune_conv_input* in, const ktune_conv_tuning* t, size_t* bytes);
/* C = op(A) op(B) on device buffers (row-major; A M x K or K x M when
 * trans_a; B K x N or N x K when trans_b; C M x N).  f32/f64: SIMT family
 * (mode selects FAST or PARITY).  bf16/f16/tf32: tcgen05 family, fp32 C. */
KTUNE_API int ktune_gemm(const ktune_gemm_input* in, const ktune_gemm_tuning* t, int mode, const void* a, const void* b,
               void* c, void* workspace, size_t workspace_bytes, void* stream);
/* Valid-mode implicit-GEMM convolution: images C,H,W,N; filters C,R,S,K;
 * outputs K,P,Q,N. */
KTUNE_API int ktune_conv(const ktune_conv_input* in, const ktune_conv_tuning* t, int mode, const void* images,
               const void* filters, void* outputs, void* workspace, size_t workspace_bytes, void* stream);

/* Host-buffer drop-ins with the executor's own contract: element counts are
 * checked like the spans of backends.cpp:237-240 ("operand size mismatch");
 * inputs are copied to the device, the kernel runs, the result is copied back
 * before return. */
KTUNE_API int ktune_execute_gemm(const ktune_gemm_input* in, const ktune_gemm_tuning* t, int mode, const void* a, int64_t a_len,
                       const void* b, int64_t b_len, void* c, int64_t c_len);
KTUNE_API int ktune_execute_conv(const ktune_conv_input* in, const ktune_conv_tuning* t, int mode, const void* images,
                       int64_t images_len, const void* filters, int64_t filters_len, void* outputs,
                       int64_t outputs_len);

/* ---- measurement (replaces CpuBackend::measure, backends.cpp:502-556) ---- */
/* require_legal under hw, seeded device operands, warm-up, best-of
 * repetitions timed with CUDA events (L2 flushed before each), returns
 * GFLOPS = 2MNK / best / 1e9 (CONV 2NPQKCRS).  opts NULL = defaults
 * {FAST, 3, 1, 1, 0x5eed}. */
KTUNE_API int ktune_measure_gemm(const ktune_hw* hw, const ktune_gemm_input* in, const ktune_gemm_tuning* t,
                       const ktune_measure_options* opts, double* gflops);
KTUNE_API int ktune_measure_conv(const ktune_hw* hw, const ktune_conv_input* in, const ktune_conv_tuning* t,
                       const ktune_measure_options* opts, double* gflops);
/* Evicts L2 with a write sweep larger than the cache (K8). */
KTUNE_API int ktune_l2_flush(void* stream);


/* ---- analytical cost model (backends.cpp:129-195; host oracle) ------------- */
KTUNE_API int ktune_peak_gflops(const ktune_hw* hw, double* out);
KTUNE_API int ktune_analytical_gflops_gemm(const ktune_hw* hw, const ktune_gemm_input* in, const ktune_gemm_tuning* t,
                                           double* out);
KTUNE_API int ktune_analytical_gflops_conv(const ktune_hw* hw, const ktune_conv_input* in, const ktune_conv_tuning* t,
                                           double* out);

/* ---- sampler (sampler.cpp:101-184); model JSON via ktune_last_text() ------- */
KTUNE_API int ktune_calibrate_gemm(const ktune_hw* hw, const ktune_gemm_input* probe, const char* bounds_json,
                                   int64_t n_uniform, uint64_t seed, double alpha);
KTUNE_API int ktune_calibrate_conv(const ktune_hw* hw, const ktune_conv_input* probe, const char* bounds_json,
                                   int64_t n_uniform, uint64_t seed, double alpha);
KTUNE_API int ktune_acceptance_rate_gemm(const ktune_hw* hw, const ktune_gemm_input* probe, const char* sampler_json,
                                         int64_t n_trials, uint64_t seed, double* rate);
KTUNE_API int ktune_uniform_acceptance_rate_gemm(const ktune_hw* hw, const ktune_gemm_input* probe,
                                                 const char* bounds_json, int64_t n_trials, uint64_t seed,
                                                 double* rate);

/* ---- input distributions (pipeline.hpp:86-118) ------------------------------ */
typedef struct ktune_gemm_distribution {
    const ktune_gemm_input* shapes; /* may be NULL when n_shapes == 0 */
    int32_t n_shapes;
    const double* weights; /* NULL = uniform over shapes */
    double fixed_fraction;
    int32_t use_ranges;
    int32_t m_lo, m_hi, n_lo, n_hi, k_lo, k_hi;
    int32_t dtype;
    int32_t randomize_transpose;
} ktune_gemm_distribution;

typedef struct ktune_conv_distribution {
    const ktune_conv_input* shapes;
    int32_t n_shapes;
    const double* weights;
    double fixed_fraction;
    int32_t use_ranges;
    int32_t n_lo, n_hi, p_lo, p_hi, q_lo, q_hi, k_lo, k_hi, c_lo, c_hi;
    const int32_t* rs_choices; /* n_rs (r, s) pairs */
    int32_t n_rs;
    int32_t dtype;
} ktune_conv_distribution;

/* ---- dataset generation (pipeline.cpp:463-556) ------------------------------ */
/* The distinct (input, tuning) sequence generate_*_dataset measures, in order
 * (the sampler RNG never depends on measurements, so it can be sharded). */
KTUNE_API int ktune_predraw_gemm(const ktune_hw* hw, const char* bounds_json, const char* sampler_json,
                                 const ktune_gemm_distribution* dist, int32_t n_samples, uint64_t seed,
                                 ktune_gemm_input* inputs_out, ktune_gemm_tuning* tunings_out, int64_t* attempts,
                                 int64_t* duplicates);
KTUNE_API int ktune_predraw_conv(const ktune_hw* hw, const char* bounds_json, const char* sampler_json,
                                 const ktune_conv_distribution* dist, int32_t n_samples, uint64_t seed,
                                 ktune_conv_input* inputs_out, ktune_conv_tuning* tunings_out, int64_t* attempts,
                                 int64_t* duplicates);
/* One rank's share of generate_gemm_dataset on the B200 backend (SURVEY
 * 8(e); reference loop pipeline.cpp:463-509).  Pre-draws the whole sequence
 * (legal draws this build cannot launch are redrawn and counted in
 * *unlaunchable), assigns indices to `world` ranks longest-processing-time
 * first by 2MNK (ktune_shard_lpt), and measures this rank's indices in
 * batches with one host sync per batch.  checkpoint_path (NULL = none):
 * every finished batch is appended; a rerun with the same arguments skips
 * the indices already recorded there.  Outputs: the full sequence
 * (inputs_out / tunings_out, n_samples entries each, may be NULL) and this
 * rank's records {index_out[i], gflops_out[i]} (cap entries; *count
 * written; gflops < 0 = launch failed).  The caller all-gathers the records
 * and rebuilds the CSV with ktune_gemm_dataset_csv. */
KTUNE_API int ktune_generate_gemm_shard(const ktune_hw* hw, const char* bounds_json, const char* sampler_json,
                                        const ktune_gemm_distribution* dist, int32_t n_samples, uint64_t seed,
                                        int32_t rank, int32_t world, const ktune_measure_options* opts,
                                        const char* checkpoint_path, ktune_gemm_input* inputs_out,
                                        ktune_gemm_tuning* tunings_out, int64_t* index_out, double* gflops_out,
                                        int64_t cap, int64_t* count, int64_t* attempts, int64_t* duplicates,
                                        int64_t* unlaunchable);
KTUNE_API int ktune_generate_conv_shard(const ktune_hw* hw, const char* bounds_json, const char* sampler_json,
                                        const ktune_conv_distribution* dist, int32_t n_samples, uint64_t seed,
                                        int32_t rank, int32_t world, const ktune_measure_options* opts,
                                        const char* checkpoint_path, ktune_conv_input* inputs_out,
                                        ktune_conv_tuning* tunings_out, int64_t* index_out, double* gflops_out,
                                        int64_t cap, int64_t* count, int64_t* attempts, int64_t* duplicates,
                                        int64_t* unlaunchable);
/* LPT assignment of n sample costs to `world` ranks: rank_out[i] = owner. */
KTUNE_API int ktune_shard_lpt(const double* costs, int64_t n, int32_t world, int32_t* rank_out);
/* Sequential generation with a backend (0 analytical, 1 b200, 2 b200-parity);
 * CSV text (pipeline.hpp:53-57 header) via ktune_last_text(). */
KTUNE_API int ktune_generate_gemm(const ktune_hw* hw, const char* bounds_json, const char* sampler_json,
                                  const ktune_gemm_distribution* dist, int32_t n_samples, uint64_t seed,
                                  int32_t backend, const ktune_measure_options* opts, int64_t* attempts,
                                  int64_t* duplicates);
/* Dataset CSV from measured records (rank 0 of a sharded run). */
KTUNE_API int ktune_gemm_dataset_csv(const ktune_gemm_input* inputs, const ktune_gemm_tuning* tunings,
                                     const double* gflops, int64_t n, const char* backend);
KTUNE_API int ktune_conv_dataset_csv(const ktune_conv_input* inputs, const ktune_conv_tuning* tunings,
                                     const double* gflops, int64_t n, const char* backend);
/* Round-trips a dataset through the loader (validation + canonical text). */
KTUNE_API int ktune_dataset_canonical(const char* csv_text, int32_t kind /* 0 gemm, 1 conv */);

/* ---- MLP performance model (perf_model.cpp) ---------------------------------- */
/* Trains on a dataset CSV on the GPU (K7); model JSON (ktune-mlp-1) via
 * ktune_last_text().  history (2 doubles per epoch: train, val MSE) may be NULL. */
KTUNE_API int ktune_mlp_train(const char* csv_text, int32_t kind, const int32_t* hidden, int32_t n_hidden,
                              int32_t log_inputs, int32_t epochs, double learning_rate, int32_t batch_size,
                              uint64_t seed, double validation_fraction, double* best_val_mse, int32_t* best_epoch,
                              double* history);
/* Glorot init (perf_model.cpp:57-79) as a model JSON. */
/* K7f: the same training (loss, shuffles, minibatches, clip, best epoch) with
 * every layer of a minibatch as one batched fp64 GEMM (GEMM summation order:
 * rounding-level differences from ktune_mlp_train). */
KTUNE_API int ktune_mlp_train_fast(const char* csv_text, int32_t kind, const int32_t* hidden, int32_t n_hidden,
                                   int32_t log_inputs, int32_t epochs, double learning_rate, int32_t batch_size,
                                   uint64_t seed, double validation_fraction, double* best_val_mse,
                                   int32_t* best_epoch, double* history);
/* The runtime candidate sweep over the whole legal space of `in` (enumerated
 * in the library, no per-candidate marshalling): fast = 0 K6 (bit-identical),
 * 1 K6f (batched GEMMs).  *device_seconds = GPU time of the sweep (K6f) or
 * the whole call (K6); *total_seconds = the whole call. */
KTUNE_API int ktune_mlp_sweep_gemm(const char* model_json, const ktune_hw* hw, const char* bounds_json,
                                   const ktune_gemm_input* in, int32_t fast, int64_t* n_candidates,
                                   double* device_seconds, double* total_seconds);
KTUNE_API int ktune_mlp_init(int32_t input_dim, const int32_t* hidden, int32_t n_hidden, int32_t log_inputs,
                             uint64_t seed, const char* feature_version);
/* GPU forward of raw feature rows (MlpModel::predict_batch, bit-exact). */
KTUNE_API int ktune_mlp_predict_rows(const char* model_json, const double* rows, int64_t n, int32_t dim, double* out);
/* GPU candidate sweep for one GEMM / CONV input (MlpPredictor::predict_*). */
/* K6f predictions (batched GEMMs, rounding-level differences from K6). */
KTUNE_API int ktune_mlp_predict_gemm_fast(const char* model_json, const ktune_gemm_input* in,
                                          const ktune_gemm_tuning* tunings, int64_t n, double* out);
KTUNE_API int ktune_mlp_predict_gemm(const char* model_json, const ktune_gemm_input* in,
                                     const ktune_gemm_tuning* tunings, int64_t n, double* out);
KTUNE_API int ktune_mlp_predict_conv(const char* model_json, const ktune_conv_input* in,
                                     const ktune_conv_tuning* tunings, int64_t n, double* out);
/* Host MSE of a model over a dataset CSV (mlp_evaluate). */
KTUNE_API int ktune_mlp_evaluate(const char* model_json, const char* csv_text, int32_t kind, double* mse);

/* ---- runtime selection (pipeline.cpp:649-723, :928-997) ---------------------- */
/* infer_*: enumerate, predict (model_json NULL = analytical oracle predictor),
 * re-measure top_k on `backend`, measured argmax; ktune-result-1 JSON via
 * ktune_last_text(). */
KTUNE_API int ktune_infer_gemm(const ktune_hw* hw, const char* bounds_json, const char* model_json,
                               const ktune_gemm_input* in, int32_t top_k, int32_t backend,
                               const ktune_measure_options* opts);
KTUNE_API int ktune_infer_conv(const ktune_hw* hw, const char* bounds_json, const char* model_json,
                               const ktune_conv_input* in, int32_t top_k, int32_t backend,
                               const ktune_measure_options* opts);
/* Sharded top-k re-measure (pipeline.cpp:674-680; with
 * top_k >= the legal space this is `bench --exhaustive`): every rank ranks
 * the same candidates and measures positions i with i % world == rank;
 * gflops_out[i] = the measurement, or -1 for another rank's position
 * (*count = candidates ranked).  After an element-wise max over ranks,
 * ktune_infer_*_replay rebuilds the ktune-result-1 JSON exactly as the
 * sequential infer_* would (ktune_last_text()). */
KTUNE_API int ktune_infer_gemm_shard(const ktune_hw* hw, const char* bounds_json, const char* model_json,
                                     const ktune_gemm_input* in, int32_t top_k, int32_t backend,
                                     const ktune_measure_options* opts, int32_t rank, int32_t world,
                                     double* gflops_out, int64_t cap, int64_t* count);
KTUNE_API int ktune_infer_conv_shard(const ktune_hw* hw, const char* bounds_json, const char* model_json,
                                     const ktune_conv_input* in, int32_t top_k, int32_t backend,
                                     const ktune_measure_options* opts, int32_t rank, int32_t world,
                                     double* gflops_out, int64_t cap, int64_t* count);
KTUNE_API int ktune_infer_gemm_replay(const ktune_hw* hw, const char* bounds_json, const char* model_json,
                                      const ktune_gemm_input* in, int32_t top_k, const char* backend_name,
                                      const double* gflops, int64_t n);
KTUNE_API int ktune_infer_conv_replay(const ktune_hw* hw, const char* bounds_json, const char* model_json,
                                      const ktune_conv_input* in, int32_t top_k, const char* backend_name,
                                      const double* gflops, int64_t n);
KTUNE_API int ktune_cache_key_gemm(const ktune_gemm_input* in);
KTUNE_API int ktune_cache_key_conv(const ktune_conv_input* in);
/* *found = 1 and the entry's JSON in ktune_last_text(), or *found = 0. */
KTUNE_API int ktune_cache_lookup_gemm(const char* dir, const ktune_gemm_input* in, int* found);
KTUNE_API int ktune_cache_lookup_conv(const char* dir, const ktune_conv_input* in, int* found);
KTUNE_API int ktune_cache_store(const char* dir, const char* result_json);
/* Runtime pick: in-memory map -> result cache (dir may be NULL) -> infer_gemm
 * on the b200 backend, storing the result; writes the chosen tuning. */
KTUNE_API int ktune_select_gemm(const ktune_hw* hw, const char* bounds_json, const char* model_json,
                                const char* cache_dir, const ktune_gemm_input* in, int32_t top_k,
                                ktune_gemm_tuning* chosen, int32_t* source /* 0 memory, 1 file, 2 inferred */);

/* Runtime pick for a convolution (infer_conv, pipeline.cpp:687-723, plus the
 * result cache :936-997): in-memory map (keyed by the input signature, hw,
 * bounds, model and top_k) -> result cache -> infer_conv on the b200 backend. */
KTUNE_API int ktune_select_conv(const ktune_hw* hw, const char* bounds_json, const char* model_json,
                                const char* cache_dir, const ktune_conv_input* in, int32_t top_k,
                                ktune_conv_tuning* chosen, int32_t* source /* 0 memory, 1 file, 2 inferred */);

/* ---- KTN1 tensor files (replaces proj/src/tensor_file.cpp:36-112) -----------
 * Same bytes as the reference writer: "KTN1", int32 element size, int32 rank,
 * int64 dims, row-major payload; f32 / f64 only (others: INVALID_ARGUMENT). */
KTUNE_API int ktune_tensor_write(const char* path, int32_t dtype, const int64_t* dims, int32_t ndims,
                                 const void* data);
/* Header into dtype / dims8[8] / ndims; the payload into data when
 * data != NULL and cap (elements) covers it (call once with data = NULL to size). */
KTUNE_API int ktune_tensor_read(const char* path, int32_t* dtype, int64_t* dims8, int32_t* ndims, void* data,
                                int64_t cap);

/* ---- command line (replaces proj/tools/ktune.cpp:700-806) ------------------
 * The `ktune` front end: argv[1] is the verb (calibrate | generate | train |
 * infer | bench | report), the flags are the reference CLI's; returns the
 * process exit code (0 success, 1 runtime failure, 2 usage error).  The
 * bin/ktune_b200 executable is a stub around this entry point. */
KTUNE_API int ktune_cli_main(int argc, char** argv);

#ifdef __cplusplus
}
#endif

#endif /* KTUNE_B200_H */
