/*
 * prnet.h -- C ABI (version 3, PRNET_ABI_VERSION) of the B200-native PRNet pattern-attention
 * forward.
 *
 * The operation (abstract, conclusion; reading fixed in
 * SURVEY.md §8(c) and restated in DESIGN.md §3): every (window b, channel c)
 * lookback series x[b][c][0..L) is cut into N = floor(L/S) segments of length
 * S (the oldest r = L - N*S points are dropped, reading A2); between every pair
 * of segments a seasonal similarity (Pearson correlation, A4) and a trend
 * distance (distance between least-squares lines normalised by the series
 * variance, A5) are evaluated; each is softmax-normalised over rows ("pattern
 * attention"; temperatures tau_s, tau_t, A6/A9) and aggregates the raw
 * segments into seasonal and trend patterns P_s, P_t (A10); a linear head over
 * the segment axis (A7/A8/A11) maps them to M = ceil(H/S) future segments, of
 * which the first H steps plus a per-step bias form y[b][c][0..H).
 *
 * Conventions for every entry point:
 *  - C linkage, no exceptions cross the boundary; every function returns a
 *    prnet_status (>= 0).  A human-readable message for the last failure is
 *    kept per handle (prnet_last_error).
 *  - Arguments are validated before any work is enqueued (SPEC-style
 *    "validate first"); on error nothing is written.
 *  - Device pointers are plain CUDA device addresses (e.g. a torch tensor's
 *    data_ptr()); host pointers are ordinary (preferably pinned) host memory.
 *  - All tensors are fp32, C-contiguous, row-major.  Sizes are int64 where they
 *    can exceed 2^31 elements (Traffic: 1.7e9 elements).
 *  - Results are deterministic: no atomics; a series' arithmetic does not
 *    depend on the batch it is in, the launch configuration or the device,
 *    so a sharded run's outputs equal the unsharded run's bitwise.
 *  - Thread safety: one handle may be used from several host threads; the
 *    last-error text is kept per handle under a lock and returned as a
 *    per-thread copy.  Stream concurrency: prnet_forward, prnet_forward_sliding
 *    and prnet_debug_* keep no per-call device state and may run concurrently
 *    on different streams with one handle (so may prnet_forward_bf16).
 *    prnet_error_sums, prnet_backward_head and prnet_backward write a per-handle
 *    device scratch buffer, and
 *    prnet_forward_host / prnet_forward_sliding_host use the handle's staging
 *    ring: calls of these on one handle must not overlap (serialise them, or
 *    use one handle per stream).
 *  - Temperatures: every tau > 0 is accepted.  The automatic kernel choice
 *    keeps each kernel inside its numerical domain: kernels that shift the
 *    seasonal logits by a known row bound need tau_seasonal >= 1/320 (tc_quad and
 *    group_f32, which shift by 1: >= 1/80); below that the row-maximum-searching FP32
 *    kernels run
 *    (warp_f32, long_f32).  A forced variant outside its domain is rejected
 *    with PRNET_ERR_UNSUPPORTED (prnet_set_kernel_variant).
 */
#ifndef PRNET_H
#define PRNET_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PRNET_ABI_VERSION 3

typedef struct prnet_handle prnet_handle; /* opaque; owned by the library */

typedef enum {
  PRNET_OK = 0,
  PRNET_ERR_INVALID_ARG = 1, /* NULL pointer with B > 0, C < 1, S < 2, L < S, H < 1,
                                tau <= 0 or non-finite, wrong parameter counts, B < 0,
                                size overflow, abi_version not in [1, 3], metric_variant
                                outside [0, 7], instance_norm not 0/1, ma_kernel not 0
                                or odd in [1, 4095]                                     */
  PRNET_ERR_BAD_STATE = 2,   /* forward before load_params; NULL handle                  */
  PRNET_ERR_UNSUPPORTED = 3, /* device is not sm_100 (cc 10.x); x/y not 16-byte aligned;
                                x and y overlap; pointer not on the handle's device;
                                shape beyond the compiled limits (N > 512; shared
                                memory of the long_f32 fallback); a forced variant
                                (prnet_set_kernel_variant) that does not cover the
                                shape, the widening flags or the seasonal temperature    */
  PRNET_ERR_CUDA = 4,        /* CUDA runtime or launch error (text: prnet_last_error)    */
  PRNET_ERR_OOM = 5          /* device or pinned-host allocation failed                  */
} prnet_status;

typedef struct {
  int32_t abi_version;      /* PRNET_ABI_VERSION (3); 1, 2 = the older layouts (ending at
                               device / instance_norm)                                    */
  int32_t channels;         /* C >= 1                                                     */
  int32_t lookback;         /* L >= seg_len                                               */
  int32_t seg_len;          /* S >= 2 (A1: S is an input, e.g. the dominant period)      */
  int32_t horizon;          /* H >= 1                                                     */
  int32_t head_per_channel; /* 1: ws/wt are [C][M][N], bias [C][H] (A7, NS "per-channel
                               linear head"); 0: one shared head [1][M][N], [1][H]       */
  int32_t metric_variant;   /* bit flags, 0 = the DESIGN.md §3 reading; SURVEY §8(f) f3:
                               bit 0 = level-only trend distance D = (mu_i - mu_j)^2;
                               bit 1 = seasonal metric on the residuals about each
                                       segment's least-squares line;
                               bit 2 = component values (A10 variant, DESIGN.md §3 R-f4):
                                       the seasonal branch aggregates z_n (bit 1: the
                                       residual z_n - kappa_n t~), the trend branch the
                                       line mu_n + kappa_n t~ (bit 0: the level mu_n)
                                       instead of the raw segments; N <= 32, M <= 32,
                                       S <= 128 (mma_f16x3) or 16 < N <= 512, S <= 96
                                       (flash_f16x3) or N <= 512 (long_f32).  Values > 7
                                       invalid.                                          */
  float tau_seasonal;       /* tau_s > 0: softmax temperature of the seasonal branch (A6) */
  float tau_trend;          /* tau_t > 0: softmax temperature of the trend branch (A6)    */
  int32_t device;           /* CUDA device ordinal the handle is bound to                 */
  /* ---- ABI 2 (a caller passing abi_version = 1 gets 0 for every field below) ---- */
  int32_t instance_norm;    /* 1 = RevIN-style normalisation of the N*S
                               segmented points (mean, population variance, eps 1e-5)
                               before the method and de-normalisation of the forecast
                               (R-f1); 0 = off                              */
  /* ---- ABI 3 (abi_version 1 or 2 callers get 0 here) ---- */
  int32_t ma_kernel;        /* 0 = off; odd k in [1, 4095] = moving-average
                               decomposition of the segmented points (edge-replicated ends,
                               after instance_norm): the seasonal branch (Def 3-4, 6, 9)
                               runs on x - MA_k(x), the trend branch (Def 3-5, 7, 9) on
                               MA_k(x) (R-f5).  Runs in mma_f16x3 (N <= 32,
                               M <= 32, S <= 128), else in long_f32 (N <= 512)            */
} prnet_config;

/* Create a handle: validates cfg, checks the device is compute capability 10.x,
 * derives N = L / S (floor), r = L - N*S, M = ceil(H / S), allocates the device
 * parameter buffers.  cfg is copied.  On error *out = NULL and the message is
 * available through prnet_last_error(NULL) (thread-local). */
prnet_status prnet_create(const prnet_config* cfg, prnet_handle** out);

/* Copy the head parameters (HOST arrays, row-major) into the handle:
 *   w_seasonal [Cw][M][N]  -- W_s[c][m][n]: weight of seasonal pattern n for
 *                             future segment m (A16: n = 0 oldest, m = 0 first)
 *   w_trend    [Cw][M][N]  -- W_t, same layout
 *   bias       [Cw][H]
 * with Cw = C if head_per_channel else 1.  n_w must equal Cw*M*N and n_b Cw*H.
 * Synchronises the handle's device before overwriting (so it may be called
 * again between forwards); the caller must not race it with in-flight work. */
prnet_status prnet_load_params(prnet_handle* h, const float* w_seasonal, const float* w_trend,
                               const float* bias, int64_t n_w, int64_t n_b);

/* Forward, DEVICE buffers: x [B][C][L] -> y [B][C][H], enqueued on cuda_stream
 * (a cudaStream_t; NULL = legacy default stream).  Asynchronous: launch errors
 * are returned, execution errors surface at the caller's next synchronisation.
 * x and y must be 16-byte aligned and must not overlap.  B = 0 is a no-op.
 * No workspace, no per-call state: concurrent forwards on different streams
 * with one handle are allowed. */
prnet_status prnet_forward(prnet_handle* h, const float* x, int64_t batch, float* y,
                           void* cuda_stream);

/* Forward, HOST buffers (end-to-end entry): x_host [B][C][L] -> y_host [B][C][H].
 * The library streams the batch through the GPU in window chunks, overlapping
 * the host->device copy of chunk k+1, the kernel on chunk k and the
 * device->host copy of chunk k-1 on its own streams, using a device staging
 * workspace it owns (allocated on first use, sized by prnet_set_host_chunk).
 * Blocking: returns after y_host is fully written.  Host buffers may be
 * pageable, but only page-locked (pinned) memory gets full PCIe bandwidth. */
prnet_status prnet_forward_host(prnet_handle* h, const float* x_host, int64_t batch,
                                float* y_host);

/* Sliding-window input mode (NS: "full sliding-window test set").
 * series: DEVICE, [C][T] fp32 row-major (channel c's T time steps contiguous),
 * 16-byte aligned.  Window b (0 <= b < batch) is x[b][c][l] = series[c][t0 + b + l],
 * l < L, so the B windows of a test set are read from C (B + L - 1) floats instead of
 * B C L.  Requires 0 <= t0 and t0 + batch - 1 + L <= T (PRNET_ERR_INVALID_ARG otherwise).
 * y: DEVICE [batch][C][H] as prnet_forward.  The result is bitwise the prnet_forward
 * result on the materialised windows.  Enqueue-only, no workspace, like prnet_forward. */
prnet_status prnet_forward_sliding(prnet_handle* h, const float* series, int64_t T,
                                   int64_t t0, int64_t batch, float* y, void* cuda_stream);

/* As prnet_forward_sliding with HOST buffers (end-to-end entry): the series span
 * [t0, t0 + batch - 1 + L) of every channel is copied to the device once (pitched),
 * then the windows are forecast in chunks whose device->host copies overlap the next
 * chunk's kernel (three streams, workspace owned by the handle).  Blocking.  Pinned
 * host memory gets full PCIe bandwidth. */
prnet_status prnet_forward_sliding_host(prnet_handle* h, const float* series, int64_t T,
                                        int64_t t0, int64_t batch, float* y_host);

/* Windows per chunk for prnet_forward_host (default: ~256 MiB of input per
 * chunk).  windows_per_chunk >= 1. */
prnet_status prnet_set_host_chunk(prnet_handle* h, int64_t windows_per_chunk);

/* Release everything the handle owns.  NULL-safe.  Caller must synchronise. */
void prnet_destroy(prnet_handle* h);

/* Message of the last failure on h (h == NULL: the calling thread's last
 * prnet_create failure).  Never NULL; valid until the next call on h. */
const char* prnet_last_error(const prnet_handle* h);

/* Derived sizes: N = floor(L/S), M = ceil(H/S), r = L - N*S. */
prnet_status prnet_get_dims(const prnet_handle* h, int32_t* N, int32_t* M, int32_t* r);

/* ---- support / debug exports (not on the timed path) ------------------- */

/* seg [B][C][N][S] (device): seg[b][c][n][t] = x[b][c][r + n*S + t]
 * (Definition step 2, reading A2).  Bit-exact gather. */
prnet_status prnet_debug_segments(prnet_handle* h, const float* x, int64_t batch, float* seg,
                                  void* cuda_stream);

/* a_s, a_t [B][C][N][N] (device): the two attention matrices, rows summing to 1, from the
 * kernel the forward runs (same arithmetic, written from the registers its fold consumes)
 * for warp_f32, mma_f16x3, tc_quad and long_f32; a handle whose forward runs small_f32 is
 * dumped by mma_f16x3, flash_f16x3 by long_f32 (same reading; every N <= 512 and every
 * widening flag).  Errors as prnet_forward; uses a stream-ordered scratch y. */
prnet_status prnet_debug_attention(prnet_handle* h, const float* x, int64_t batch, float* a_s,
                                   float* a_t, void* cuda_stream);

/* out3 (device, 3 doubles) = {sum (y - target)^2, sum |y - target|, count} over
 * n = batch*C*H elements, fp64, fixed reduction order (deterministic).  The
 * per-rank input of the NCCL all-reduce that forms MSE / MAE. */
prnet_status prnet_error_sums(prnet_handle* h, const float* y, const float* target,
                              int64_t batch, double* out3, void* cuda_stream);

/* Backward pass of the head (DESIGN.md §3 reading R-f6): the gradients of
 * L = sum(dy * y) with respect to w_seasonal, w_trend and bias, for the forward of x:
 *   dws[cw][m][n] = sum_{b, c -> cw, t} dY[m][t] P_s[n][t],  dwt likewise with P_t,
 *   db[cw][h] = sum_{b, c -> cw} dy[b][c][h] s_r,   dY[m][t] = dy[b][c][m S + t] s_r,
 * where P_s, P_t are the series' patterns (Def 9, after instance normalisation when on),
 * s_r the instance-normalisation scale (1 when off), and c -> cw the head of channel c
 * (all channels -> 0 for a shared head).  The gradients do not depend on the loaded head, so
 * prnet_load_params is not required.
 *   x   device [B][C][L] fp32 (as prnet_forward);  dy  device [B][C][H] fp32
 *   dws, dwt  device [Cw][M][N] fp32, db device [Cw][H] fp32: overwritten (B = 0 -> zeros)
 * FP32 recomputation of the attention, fixed-order reductions (fp64 across CTAs): the result
 * is deterministic.  Uses a per-handle device workspace (grown on demand, which synchronises
 * the stream once).  N <= 32 (S <= 128): one warp per series; N > 32 or S > 128: one CTA
 * per series, rows streamed.  Errors: INVALID_ARG (B < 0, NULL pointers), UNSUPPORTED
 * (N > 512, M > 32, metric_variant bit 2, ma_kernel > 0, pointers not on the handle's
 * device), CUDA, OOM. */
prnet_status prnet_backward_head(prnet_handle* h, const float* x, int64_t batch,
                                 const float* dy, float* dws, float* dwt, float* db,
                                 void* cuda_stream);

/* the forward with x [B][C][L] and y [B][C][H] as bf16 bit patterns
 * (device, uint16_t; half the HBM bytes of prnet_forward).  The values are widened to fp32
 * exactly and every step runs as in prnet_forward's S = 24 tc_quad kernel; y is rounded to the
 * nearest bf16 (ties to even) at the store.  Needs the S = 24 tc_quad domain (N <= 32,
 * M <= 32, tau_seasonal >= 1/80) and the base reading (metric_variant 0, no instance_norm, no
 * ma_kernel).  x, y 4-byte aligned (16 bytes, L % 8 == 0, r % 8 == 0: one bulk copy per
 * series), not overlapping.  Errors as prnet_forward; UNSUPPORTED outside that domain. */
prnet_status prnet_forward_bf16(prnet_handle* h, const uint16_t* x, int64_t batch, uint16_t* y,
                                void* cuda_stream);

/* SURVEY §8(f) f4, the full backward (reading R-f7 in DESIGN.md §3): for the upstream
 * gradient dy = dL/dy [B][C][H] (device, fp32) of one forward over x [B][C][L], writes
 *   dx   [B][C][L]   dL/dx (0 at the r dropped oldest points of each window),
 *   dws, dwt [Cw][M][N], db [Cw][H]   the head gradients, summed over the batch (and over the
 *                     channels for a shared head), as prnet_backward_head,
 *   dtau [2]          dL/dtau_seasonal, dL/dtau_trend, summed over every series,
 * all device fp32, overwritten (B = 0: zero head / temperature gradients).  The attention is
 * recomputed in FP32 (row maxima searched: every tau > 0), each step the adjoint of one
 * Definition step; deterministic (fixed-order reductions, no atomics).  Uses the per-handle
 * device workspace of prnet_backward_head (not stream-concurrent on one handle).  Base reading
 * only.  Errors: BAD_STATE (before load_params), INVALID_ARG (B < 0, NULL pointers),
 * UNSUPPORTED (N > 32, M > 32, S > 128, metric_variant bits 1-2, instance_norm, ma_kernel,
 * pointers not on the handle's device), CUDA, OOM. */
prnet_status prnet_backward(prnet_handle* h, const float* x, int64_t batch, const float* dy,
                            float* dx, float* dws, float* dwt, float* db, float* dtau,
                            void* cuda_stream);

/* Select the forward kernel (tuning / cross-checking; default -1 = automatic).
 * All variants compute the same reading to within the documented tolerance:
 *   0 = warp_f32     one warp per series, CUDA-core FP32                  (N <= 32)
 *                    [auto: fallback, e.g. S > 128 or tau_seasonal < 1/320]
 *   1 = long_f32     one CTA per series, rows streamed, FP32              (N <= 512)
 *                    [auto: N > 32 when neither 5 nor 8 applies]
 *   2 = mma_f16x3    one warp per series, mma.sync m16n8k16 with split-fp16
 *                    hi/lo operands, 3 products, fp32 accumulation
 *                    (N <= 32, M <= 32, S <= 128)  [auto: N <= 32 unless 6, 7, 9 apply]
 *   3, 4             retired (round-1 tcgen05 prototypes, superseded by 6):
 *                    PRNET_ERR_INVALID_ARG
 *   5 = flash_f16x3  one CTA per series, 16-key tiles streamed, mma.sync
 *                    split-fp16 (16 < N <= 512, S <= 96, M <= 32)  [auto: N > 32 unless 8]
 *   6 = tc_quad      groups of 4 warps take quads of 4 series; Gram of the
 *                    row-normalised segments and the fold on tcgen05 / TMEM,
 *                    head on per-warp mma.sync (split fp16), lane-per-row
 *                    softmaxes (S in {12, 16, 24, 32, 48, 64, 96}, N <= 32,
 *                    M <= 32 for S = 24 else M <= 64, tau_seasonal >= 1/80;
 *                    S = 24 also takes metric_variant bits 1-2 and instance_norm,
 *                    not ma_kernel)  [auto: N > 16; S = 48 with N > 8; M > 32;
 *                    S = 24 with the widening for N > 8]
 *   7 = small_f32    one warp per series with lanes over TIME, FP32, warp
 *                    butterfly reductions (N <= 16, S <= 128, M <= 32)
 *                    [auto: N <= 8 or S > 64 where 9 does not apply]
 *   8 = tc_long      one CTA (16 softmax warps + 1 MMA warp) per series; 128-row query
 *                    x 64-key tiles: Gram and P = E X' on tcgen05 / TMEM, exponentials
 *                    in TMEM, head on mma.sync (32 < N <= 512, S in {12, 24, 48, 96},
 *                    M <= 64, tau_seasonal >= 1/16, plain reading)
 *                    [auto: S >= 48 with N >= 200; M <= 8 with S = 12, N >= 100 or
 *                    S = 24, N >= 200; M > 32]
 *   9 = group_f32    lanes over (series, segment), 32 / NP series per warp, FP32
 *                    (N <= 16, S <= 32, tau_seasonal >= 1/80)
 *                    [auto: N <= 8, S <= 16 or M > 32]
 * Variants 2, 5, 7 need tau_seasonal >= 1/320 (known-maximum softmax shift), 8 needs
 * tau_seasonal >= 1/16 (its fp16 E operand, DESIGN.md R-tcl); 6 and 9 tau_seasonal >= 1/80
 * (the symmetric shift 1); below the floors the automatic choice is 0 (N <= 32, no
 * widening) or 1.
 * Returns PRNET_ERR_UNSUPPORTED when the variant does not cover the handle's shape. */
prnet_status prnet_set_kernel_variant(prnet_handle* h, int32_t variant);

/* Kernel-level accounting for the bench (host-side, no device work):
 * kernel_launches = device kernels one prnet_forward(batch) enqueues. */
prnet_status prnet_forward_plan(const prnet_handle* h, int64_t batch, int32_t* kernel_launches,
                                int32_t* variant);  /* variant as above */

#ifdef __cplusplus
}
#endif
#endif /* PRNET_H */
