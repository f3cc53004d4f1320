/*
 * tbgpu.h — C ABI of the B200-native FP64 square-GEMM hot path
 * (arXiv 2509.04594 "hand-rolled CUDA" tiled DGEMM, C = A·B).
 *
 * Drop-in boundary. The reference's binding surface for this path is the flat
 * foreign-function-shaped entry of its GPU package,
 *     gpuTiledMultiplyFlat(device, a, b, m, k, n, tileEdge, outC, outSeconds) -> status
 *     (/root/reference/pkg/gpu/src/multiply.ts:54-79, status codes :49-52;
 *      SPEC.md:453 "flat C-style interface ... out-parameters for result
 *      buffer and device seconds"),
 * registered into the Python harness as the `MultiplyFn` backend
 * "gpu-tiled" (backends.py:56, :270-272; registry.ts:58-71).
 * Every function below names the reference interface it replaces.
 *
 * Conventions
 *  - All matrices are row-major float64 ("C-contiguous", matrices.py:1-5):
 *    A is m x k (leading dim lda >= k), B is k x n (ldb >= n), C is m x n
 *    (ldc >= n). C is fully overwritten unless `accumulate` is set.
 *  - Device pointers (tb_dgemm*, tb_cublas_dgemm) come from the caller (in
 *    this repo: torch CUDA tensors' data_ptr()); the library never allocates
 *    caller-visible memory. Host pointers (tb_gpu_tiled_multiply_flat*) are
 *    plain host buffers; the library stages them through a per-device cached
 *    workspace, exactly as the reference executor copies to "device" buffers
 *    before its kernel clock starts (executor.ts:92-104).
 *  - Kernel seconds are kernel-only device time from CUDA events recorded on
 *    the launching stream (executor.ts:104,144).
 *  - Returns a TB_STATUS_* code; never throws, never aborts. On status != 0,
 *    tb_last_error() gives a thread-local message.
 */
#ifndef TBGPU_H_
#define TBGPU_H_

#include <stdint.h>

#if defined(__GNUC__)
#define TB_API __attribute__((visibility("default")))
#else
#define TB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes — multiply.ts:49-52 (0..3) plus 4 for CUDA/NCCL runtime errors. */
#define TB_STATUS_OK 0
#define TB_STATUS_BAD_DIMS 1
#define TB_STATUS_OVER_LIMITS 2
#define TB_STATUS_NO_DEVICE 3
#define TB_STATUS_RUNTIME 4

/* Kernel variants. AUTO picks DMMA_TMA when the TMA alignment rules hold
 * (16-byte aligned bases and leading dims, i.e. even lda/ldb for float64)
 * and DMMA_CPASYNC otherwise. PAPER is a faithful CUDA restatement of the
 * reference's tiledKernelThread (kernel.ts:50-78): tile_edge x tile_edge
 * threads, two shared tiles, running sum in k order, no FMA contraction —
 * bitwise equal to the reference's naive oracle. */
#define TB_VARIANT_AUTO 0
#define TB_VARIANT_PAPER 1
#define TB_VARIANT_DMMA_TMA 2
#define TB_VARIANT_DMMA_CPASYNC 3
#define TB_VARIANT_DFMA 4 /* same pipeline/schedule, scalar DFMA 8x8 register tiles (comparison path) */
#define TB_NUM_VARIANTS 5

#define TB_DEFAULT_TILE_EDGE 32 /* limits.ts:40-42 */

/* Replaces gpuTiledMultiplyFlat (multiply.ts:54-79) one for one: host
 * buffers in, caller-owned outC (length out_c_len, must equal m*n, else
 * BAD_DIMS as at multiply.ts:66) and outSeconds (kernel-only seconds).
 * device < 0 or no CUDA device -> TB_STATUS_NO_DEVICE (multiply.ts:65).
 * tile_edge follows validateLaunch (limits.ts:58-79): < 1 -> BAD_DIMS,
 * tile_edge^2 > 1024 threads -> OVER_LIMITS. Uses TB_VARIANT_AUTO. */
TB_API int tb_gpu_tiled_multiply_flat(int32_t device, const double* a, const double* b,
                               int64_t m, int64_t k, int64_t n, int32_t tile_edge,
                               double* out_c, int64_t out_c_len, double* out_seconds);

/* Same as above with an explicit variant and an optional end-to-end clock:
 * out_e2e_seconds (nullable) receives device time from the first H2D copy to
 * the end of the last D2H copy (the `e2e` bench leg). Large calls run a
 * copy/compute pipeline (shape: tb_pipeline_plan);
 * out_seconds is then the union of the GEMM launches' intervals.
 * With pageable a or b (staged through pinned slots) on a large call (fused
 * phase 1, >= 2e11 flops), the phase-1 kernel waits on copies this thread
 * enqueues over the call: other threads should not issue device-synchronising
 * calls (cudaFreeHost, cudaFree, ...) on the same device meanwhile. If one
 * blocks the enqueue for longer than the flag-wait timeout (10 s;
 * TB_PIPE_TIMEOUT_MS), the kernel aborts cleanly: the call returns
 * TB_STATUS_RUNTIME (tb_last_error names the panel), out_c is not valid, and
 * the CUDA context stays usable. Pinned buffers have no such window.
 * out_seconds on the fused path is the union of the GEMM launch spans; the
 * phase-1 launch's span includes its waits for panels still in flight, so it
 * can exceed pure compute time when the copies lag (it is "kernel-only" in
 * the reference's sense: no launch, copy or sync outside a kernel). */
TB_API int tb_gpu_tiled_multiply_flat_ex(int32_t device, const double* a, const double* b,
                                  int64_t m, int64_t k, int64_t n, int32_t tile_edge,
                                  int32_t variant, double* out_c, int64_t out_c_len,
                                  double* out_seconds, double* out_e2e_seconds);

/* Device-pointer form used by the Python MultiplyFn backend (the "gpu-tiled"
 * registration, registry.ts:58-71 / backends.py:270-272): synchronous,
 * kernel-only seconds from events on `cuda_stream` (a cudaStream_t; NULL =
 * legacy default stream). Square or rectangular, packed leading dims. */
TB_API int tb_dgemm(const double* A, const double* B, double* C, int64_t m, int64_t k, int64_t n,
             int32_t tile_edge, int32_t variant, int32_t device, void* cuda_stream,
             double* out_kernel_seconds);

/* Asynchronous launch with explicit leading dims and C += A·B when
 * `accumulate` != 0 (the K-panel step of the row-sharded multi-GPU driver,
 * SURVEY.md §8(e)). No synchronisation, no timing; errors from the launch
 * itself are reported. Runs on the current device. */
TB_API int tb_dgemm_launch(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                    int64_t ldc, int64_t m, int64_t k, int64_t n, int32_t accumulate,
                    int32_t tile_edge, int32_t variant, void* cuda_stream);

/* cuBLAS DGEMM baseline (the paper's CuBLAS row; SPEC.md:15
 * external registration) with the tb_dgemm signature; variant/tile ignored.
 * Native FP64 (no emulation API exists for DGEMM in this toolkit). */
TB_API int tb_cublas_dgemm(const double* A, const double* B, double* C, int64_t m, int64_t k,
                    int64_t n, int32_t tile_edge, int32_t variant, int32_t device,
                    void* cuda_stream, double* out_kernel_seconds);

/* EXPERIMENTAL — not a measured path. The measured multi-GPU path is one
 * process per GPU with an NCCL broadcast of B (multigpu.ShardedGemm, device
 * buffers; multigpu.HostShardedGemm from host buffers; bench.py --gpus N),
 * as BASELINE.json's north_star specifies. This single-process peer-copy
 * form is kept for callers that drive several GPUs from one thread; it is
 * tested for parity with a device listed several times, never on distinct
 * GPUs.
 *
 * Row-sharded multi-GPU GEMM from one process (the
 * reference's multi-device row partition is plan_partitions,
 * backends.py:119-136). Entry i of `devices` owns rows[i] rows:
 * C_rows[i] (rows[i] x n) = A_rows[i] (rows[i] x k) · B, all packed
 * row-major on devices[i]; rows[i] may be 0. B_root (k x n) is on
 * devices[0]; B_replicas[i] (k x n, i >= 1) receives B on devices[i]
 * (entry 0 unused; the table may be NULL when ndev == 1). B is forwarded
 * in K-panels down the chain devices[0] -> devices[1] -> ... by peer copies
 * overlapped with each device's panel GEMMs. A device may appear more than
 * once (tests). The caller's buffers must be ready before the call (it does
 * not order itself after the caller's streams); synchronous.
 * out_kernel_seconds_max: max over devices of first-GEMM start .. last-GEMM
 * end (CUDA events); out_total_seconds (nullable): host clock around the
 * whole exchange + compute. variant: AUTO / DMMA_* / DFMA (not PAPER).
 * No communicator handle (the tb_mgpu_init / tb_mgpu_destroy pair SURVEY.md
 * §8(b) sketches): the exchange is peer copies on the library's per-device
 * streams, so there is no NCCL state to own; tb_release frees the streams. */
TB_API int tb_dgemm_mgpu(int32_t ndev, const int32_t* devices, const double* const* A_rows,
                         const double* B_root, double* const* B_replicas, double* const* C_rows,
                         const int64_t* rows, int64_t k, int64_t n, int32_t variant,
                         double* out_kernel_seconds_max, double* out_total_seconds);

/* Asynchronous 2D copy (cudaMemcpy2DAsync, direction inferred from the
 * pointers): `rows` rows of `width_bytes` from src (pitch spitch_bytes) to dst
 * (pitch dpitch_bytes) on `cuda_stream`. Plumbing for the host-buffer
 * multi-GPU driver (multigpu.HostShardedGemm uploads A[:, k-panel] slices
 * from pinned memory without a host-side gather); no reference counterpart. */
TB_API int tb_copy2d_async(void* dst, int64_t dpitch_bytes, const void* src, int64_t spitch_bytes,
                           int64_t width_bytes, int64_t rows, void* cuda_stream);

/* Launch validation only (limits.ts:58-79 validateLaunch), no device work
 * beyond attribute queries: returns the status tb_dgemm would return for
 * these arguments before launching. */
TB_API int tb_validate_launch(int64_t m, int64_t k, int64_t n, int32_t tile_edge, int32_t variant,
                       int32_t device);

/* Number of CUDA devices (0 when there is no driver / device) —
 * probeDevice() (executor.ts:158-162). */
TB_API int tb_device_count(void);

/* Variant name ("paper", "dmma_tma", ...) or NULL when out of range. */
TB_API const char* tb_variant_name(int32_t variant);

/* The variant AUTO resolves to for these arguments (-1 on bad args). */
TB_API int tb_resolve_variant(const void* A, int64_t lda, const void* B, int64_t ldb, int32_t variant);

/* Thread-local message for the last failing call on this thread. */
TB_API const char* tb_last_error(void);

/* Library version string. */
TB_API const char* tb_version(void);

/* The host-buffer pipeline's shape for an m x k x n call on a device with
 * `sms` SMs (no device work; tests and tooling); `staging` bit 0: A or B is
 * pageable (staged through pinned slots), bit 1: C is pageable: phase-1 rows *out_mq, whether
 * phase 1 runs as the fused flag-driven launch, the K-panel bounds
 * out_panels[0..*out_npanels) (0 .. k) and the phase-2 row-block bounds
 * out_blocks[0..*out_nblocks) (*out_mq .. m). OVER_LIMITS (counts still set)
 * when the arrays are too small. Internal to tb_gpu_tiled_multiply_flat_ex;
 * no reference counterpart. */
TB_API int tb_pipeline_plan(int64_t m, int64_t k, int64_t n, int32_t sms, int32_t fused_ok,
                            int32_t staging, int64_t* out_mq,
                            int32_t* out_fused, int64_t* out_panels, int32_t max_panels, int32_t* out_npanels,
                            int64_t* out_blocks, int32_t max_blocks, int32_t* out_nblocks);

/* Number of kernels this library has launched so far in this process (its
 * own GEMM, strip, pipeline and staging kernels; not cuBLAS). */
TB_API long long tb_kernel_launches(void);

/* Run metadata (the reference's RunMetadata.capture hook, harness.py:126-142;
 * SURVEY.md §5 "Metrics / logging") as one JSON object in buf (NUL
 * terminated): this library's version and path, CUDA runtime / driver
 * versions, the cuBLAS actually loaded (runtime version and file path — in a
 * process that imported torch first it is torch's copy), its pinned math
 * mode and FP64 emulation state, and for `device` (if present) the GPU name,
 * SM count, compute capability, L2 / HBM size and max clocks.
 * OVER_LIMITS when buf_len is too small. */
TB_API int tb_runtime_info(int32_t device, char* buf, int64_t buf_len);

/* The launches tb_dgemm would enqueue for a packed, 16-byte aligned
 * m x k x n product on a device with `sms` SMs (no device work): a JSON array
 * with, per launch, the kernel (dmma / dfma / paper), loader, CTA tile,
 * sub-problem shape, grid and persistent schedule (data-parallel / stream-K /
 * split-K shape, tiles, k-iterations per CTA, segments) and whether it is an
 * edge strip. The "resolved variant / tile" of the run metadata. */
TB_API int tb_launch_plan(int64_t m, int64_t k, int64_t n, int32_t variant, int32_t sms, char* buf,
                          int64_t buf_len);

/* Free the cached host-entry workspaces and cuBLAS handles. */
TB_API void tb_release(void);

#ifdef __cplusplus
}
#endif

#endif /* TBGPU_H_ */
