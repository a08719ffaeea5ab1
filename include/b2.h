/*
 * libb2 — B200-native executor for MLModelCI's profiling hot path (C ABI).
 *
 * This is the drop-in boundary between the reference's Python control plane
 * (register / convert / profile) and hand-written sm_100a kernels.  Plain
 * pointers and sizes only; no torch or CUDA types in the signatures
 * (cudaStream_t travels as void*).
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/pkg/src/modelci/):
 *
 *   b2_plan_create   MockServer.__init__ model load        mockserve/server.py:94-109
 *                    + toyformat.load_model / model_dims  converter/toyformat.py:152-162
 *   b2_plan_io       toyformat.model_dims (in/out dims)     converter/toyformat.py:159-162
 *   b2_forward       MockServer.predict (device buffers)    mockserve/server.py:117-127
 *   b2_forward_host  MockServer.predict as the RPC path sees it: host batch in,
 *                    host outputs back (H2D + forward + D2H) mockserve/server.py:169-180,216-241
 *   b2_bench         measure_cell's closed-loop timing loop profiler/clients.py:161-255
 *                    (hot loop :217-231) -> per-request latency + completion ms,
 *                    the LatencySamples fields of profiler/stats.py:21-38
 *   b2_gen_input     build_payload (synthetic request bodies) profiler/clients.py:153-158
 *   b2_plan_memory   ProcessStatsReader.read's memory figure for the instance
 *                    (RSS there, device bytes here)          telemetry/providers.py:147-170
 *   b2_plan_destroy  MockServer.shutdown                    mockserve/server.py:132-134
 *   b2_last_error    the exception text the reference raises (ToyFormatError,
 *                    RequestFailure, ...) errors.py
 *
 * Threading: a plan is bound to the device current at creation and is not
 * thread-safe; callers serialise calls per plan (the worker holds a lock,
 * matching the reference's one-request-per-connection model).
 */
#ifndef B2_H
#define B2_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define B2_API __attribute__((visibility("default")))
#else
#define B2_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (0 = OK); runtime.py maps them onto errors.py classes */
#define B2_OK 0
#define B2_ERR_FORMAT 1      /* malformed plan blob           -> PlanFormatError    */
#define B2_ERR_UNSUPPORTED 2 /* op/shape the kernels lack      -> PlanFormatError    */
#define B2_ERR_CUDA 3        /* CUDA runtime/launch failure    -> LaunchFailure/CellFailure */
#define B2_ERR_ARG 4         /* bad argument (batch < 1, NULL) -> InvalidRequest     */
#define B2_ERR_NODEVICE 5    /* no CUDA device visible         -> LaunchFailure      */
#define B2_ERR_FUSED 6       /* b2_read_tensor: intermediate fused into its consumer,
                                never materialised (verification hook only)        */

/* execution dtypes */
#define B2_DT_FROM_PLAN -1
#define B2_DT_FP32 0
#define B2_DT_BF16 1

/* input kinds reported by b2_plan_io */
#define B2_IN_DENSE_F32 0
#define B2_IN_TOKENS_I64 1

typedef struct b2_plan b2_plan;

/* Parse a b200-plan blob, upload weights in kernel layouts (bf16 K-major
 * tiles for tcgen05, or fp32), and bind the plan to the current device. */
B2_API int b2_plan_create(const void* blob, size_t len, int dtype, b2_plan** out);

/* Per-sample element counts and the input element type. */
B2_API int b2_plan_io(const b2_plan* plan, int64_t* in_elems_per_sample, int* in_kind,
               int64_t* out_elems_per_sample);

/* Model facts: algorithmic FLOPs per sample, weight bytes resident in HBM,
 * number of kernel launches one forward issues. */
B2_API int b2_plan_info(const b2_plan* plan, double* flops_per_sample, double* weight_bytes,
                 int* launches_per_forward, int* dtype);

/* One forward on device buffers: d_in [batch, in_elems] (f32 or i64),
 * d_out [batch, out_elems] f32.  Enqueued on `stream` (NULL = the plan's
 * stream); the call does not synchronise. */
B2_API int b2_forward(b2_plan* plan, const void* d_in, void* d_out, int batch, void* stream);

/* Host buffers in and out: H2D copy, forward, D2H copy, synchronised. */
B2_API int b2_forward_host(b2_plan* plan, const void* h_in, void* h_out, int batch);

/* Closed-loop device-timed measurement of one sweep cell: `warmup` untimed
 * forwards then `n` timed ones on device-resident seeded inputs, each replayed
 * from a CUDA graph and bracketed by CUDA events.  lat_ms[i] is request i's
 * device time, completion_ms[i] its completion instant since the first
 * request started (host arrays of n floats). */
B2_API int b2_bench(b2_plan* plan, int batch, int warmup, int n, uint64_t seed, float* lat_ms,
             float* completion_ms);

/* Same loop but every request goes host->device->host through pinned buffers
 * (the end-to-end view a remote client sees); inputs regenerated per seed. */
B2_API int b2_bench_e2e(b2_plan* plan, int batch, int warmup, int n, uint64_t seed, float* lat_ms,
                 float* completion_ms);

/* Seeded synthetic inputs written to a device buffer (N(0,1) f32 or uniform
 * token ids) — the device-side build_payload. */
B2_API int b2_gen_input(b2_plan* plan, void* d_in, int batch, uint64_t seed, void* stream);

/* Per-op device times (ms) of one forward at `batch`, averaged over `iters`
 * eager runs: op_ms[i] for op i (n_ops entries; returns the count in *n_ops). */
B2_API int b2_profile_ops(b2_plan* plan, int batch, int iters, float* op_ms, int* n_ops,
                   int* op_kinds);

/* Copy activation tensor `tensor` (as stored: bf16/fp32, or int32 ids) of the
 * last forward run at `batch` into host memory (verification hook: lets the
 * parity tests check every op against the oracle on the kernel's own inputs).
 * Returns B2_ERR_FUSED for intermediates the executor never materialises
 * (the stem output under the fused stem/max-pool, a ResNet projection
 * shortcut folded into its block's last conv). */
B2_API int b2_read_tensor(b2_plan* plan, int batch, int tensor, void* host_out, size_t bytes);

/* Device memory the plan holds right now (weights, per-batch activation
 * arenas, I/O buffers, split-K workspaces): the instance's memory indicator
 * of a profiled cell (ProfilingResult.memory_bytes). */
B2_API int b2_plan_memory(const b2_plan* plan, uint64_t* device_bytes);

B2_API void b2_plan_destroy(b2_plan* plan);

/* Thread-local message for the last nonzero status. */
B2_API const char* b2_last_error(void);

/* Library build string (arch, git-free version). */
B2_API const char* b2_version(void);

#ifdef __cplusplus
}
#endif
#endif /* B2_H */
