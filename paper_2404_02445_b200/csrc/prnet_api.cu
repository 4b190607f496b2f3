// prnet_api.cu -- the C ABI of include/prnet.h: validation, handle state,
// kernel-variant selection, and the host-buffer streaming runtime
// (prnet_forward_host).  No torch types, no exceptions across the boundary.
#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/prnet.h"
#include "prnet_internal.cuh"

struct prnet_handle {
  prnet_config cfg;
  int N, r, M, Cw;
  int sm_count, max_smem_optin;
  float* d_ws = nullptr;
  float* d_wt = nullptr;
  float* d_b = nullptr;
  double* d_err = nullptr;  // error-sum partials
  unsigned char* d_wpack = nullptr;  // mma variant: packed fp16 hi/lo head
  float* d_invsw = nullptr;
  unsigned char* d_wpack_tc = nullptr;  // tc variant: head as the tcgen05 B operand
  unsigned char* d_wpack_fl = nullptr;  // flash variant: head [16 MMT][2 Npad] hi/lo
  float* d_invsw_fl = nullptr;
  bool loaded = false;
  int forced_variant = -1;  // prnet_set_kernel_variant
  mutable std::mutex err_mu;   // err is written by any thread that calls into the handle
  std::string err;
  // host-forward runtime
  int64_t host_chunk = 0;   // windows per chunk (0 = default)
  int64_t stage_windows = 0;    // windows the x staging ring holds
  int64_t ystage_windows = 0;   // windows the y staging ring holds
  static constexpr int kStages = 3;
  float* d_xstage[kStages] = {nullptr, nullptr, nullptr};
  float* d_ystage[kStages] = {nullptr, nullptr, nullptr};
  cudaStream_t streams[kStages] = {nullptr, nullptr, nullptr};
  float* d_series = nullptr;   // prnet_forward_sliding_host: device copy of the series span
  int64_t series_floats = 0;
  float* d_bwd = nullptr;      // prnet_backward_head: per-CTA partials
  int64_t bwd_floats = 0;
};

namespace {

thread_local std::string g_create_error;

prnet_status fail(prnet_handle* h, prnet_status s, const std::string& msg) {
  if (h) {
    std::lock_guard<std::mutex> lk(h->err_mu);
    h->err = msg;
  } else {
    g_create_error = msg;
  }
  return s;
}

prnet_status cuda_fail(prnet_handle* h, cudaError_t e, const char* what) {
  std::string m = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
                  ")";
  return fail(h, e == cudaErrorMemoryAllocation ? PRNET_ERR_OOM : PRNET_ERR_CUDA, m);
}

// RAII device switch (the caller's current device is restored).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    if (cudaGetDevice(&cur) == cudaSuccess && prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

prnet::FwdArgs make_args(const prnet_handle* h, const float* x, int64_t B, float* y) {
  prnet::FwdArgs a{};
  const prnet_config& c = h->cfg;
  a.x = x;
  a.y = y;
  a.ws = h->d_ws;
  a.wt = h->d_wt;
  a.bias = h->d_b;
  a.wpack = reinterpret_cast<const uint4*>(h->d_wpack);
  a.wpack_inv_sw = h->d_invsw;
  a.wpack_tc = reinterpret_cast<const uint4*>(h->d_wpack_tc);
  a.wpack_flash = h->d_wpack_fl;
  a.wpack_flash_inv_sw = h->d_invsw_fl;
  a.B = B;
  a.xsb = (int64_t)c.channels * c.lookback;   // [B][C][L]; prnet_forward_sliding overrides
  a.xsc = c.lookback;
  a.x_vec = ((c.lookback & 3) == 0) && ((h->r & 3) == 0);
  a.C = c.channels;
  a.L = c.lookback;
  a.S = c.seg_len;
  a.H = c.horizon;
  a.N = h->N;
  a.r = h->r;
  a.M = h->M;
  a.head_per_channel = c.head_per_channel ? 1 : 0;
  a.ks = prnet::kLog2e / c.tau_seasonal;
  a.kt = prnet::kLog2e / c.tau_trend;
  const double S = c.seg_len;
  a.half_s = (float)(0.5 * (S - 1.0));
  a.inv_v = (float)(12.0 / (S * (S * S - 1.0)));
  // metric_variant bit 0 (level-only trend): the kappa term of Def 7 drops
  a.vtrend = (c.metric_variant & 1) ? 0.f : (float)((S * S - 1.0) / 12.0);
  a.detrend = (c.metric_variant >> 1) & 1;
  a.revin = c.instance_norm;
  a.comp = (c.metric_variant >> 2) & 1;
  a.ma_k = c.ma_kernel;
  a.ma_inv = c.ma_kernel > 0 ? 1.0f / (float)c.ma_kernel : 0.f;
  a.inv_s = (float)(1.0 / S);
  a.inv_n = (float)(1.0 / h->N);
  a.inv_ns = (float)(1.0 / ((double)h->N * S));
  return a;
}

// Checks a device pointer lives on the handle's device.
prnet_status check_dev_ptr(prnet_handle* h, const void* p, const char* name) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(h, PRNET_ERR_UNSUPPORTED, std::string(name) + " is not a CUDA pointer");
  }
  if (!(at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) ||
      at.device != h->cfg.device)
    return fail(h, PRNET_ERR_UNSUPPORTED,
                std::string(name) + " is not device memory on device " +
                    std::to_string(h->cfg.device));
  return PRNET_OK;
}

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  uintptr_t pa = (uintptr_t)a, pb = (uintptr_t)b;
  return pa < pb + nb && pb < pa + na;
}

// 0 = warp_f32 (N <= 32, CUDA-core FP32), 1 = long_f32 (32 < N <= 512),
// 2 = mma_f16x3 (N <= 32, M <= 32: mma.sync tensor cores, split-fp16 3-product),
// 3, 4 = retired (round-1 tcgen05 prototypes tc_fold / tc_full, superseded by 6).
// 5 = flash_f16x3 (16 < N <= 512, S <= 96, M <= 32: key-streaming mma.sync, long lookbacks)
bool flash_applicable(const prnet_handle* h) {
  return h->N > 16 && h->N <= 512 && h->cfg.seg_len <= 96 && h->M <= 32;
}
// the tcgen05 head tile (pack_tc_head) is packed for every N <= 32, M <= 32 handle with a
// tc_quad instantiation (S = 24: fwd_tcq.cu; S in {12, 16, 32, 48, 64, 96}: fwd_tcg.cu)
bool tc_head_shape(const prnet_handle* h) {
  if (h->N > 32) return false;
  if (h->cfg.seg_len == 24) return h->M <= 32;
  return prnet::tcg_supported_s(h->cfg.seg_len) && h->M <= 64;   // fwd_tcg.cu: M <= 64
}
// 6 = tc_quad (S = 24, N <= 32, M <= 32, tau_s >= 1/80: quads of series on tcgen05 / TMEM,
// seasonal shift 1 >= rho keeps the diagonal term normal only down to tau_s = 1/80)
bool tcq_applicable(const prnet_handle* h) {
  return tc_head_shape(h) && h->cfg.tau_seasonal >= 0.0125f;
}
// the widening flags are compiled into the S = 24 kernel only (its WIDE instantiation)
bool tcq_wide_applicable(const prnet_handle* h) {
  return tcq_applicable(h) && h->cfg.seg_len == 24;
}
// Variants that implement the SURVEY §8(f) widening: the level-only trend runs in every
// kernel (a.vtrend = 0); the detrended seasonal metric and instance normalisation in
// tc_quad, mma_f16x3 (N <= 32) and flash_f16x3 (16 < N <= 512, S <= 96); component values
// (bit 2) in mma_f16x3, tc_quad (S = 24), flash_f16x3 and long_f32.
bool widening_on(const prnet_handle* h) {
  return (h->cfg.metric_variant & 6) != 0 || h->cfg.instance_norm != 0 || h->cfg.ma_kernel > 0;
}
// component values: mma_f16x3, flash_f16x3, long_f32; the moving-average decomposition:
// mma_f16x3 (N <= 32), long_f32
bool comp_on(const prnet_handle* h) {
  return (h->cfg.metric_variant & 4) != 0 || h->cfg.ma_kernel > 0;
}
bool variant_supports_widening(const prnet_handle* h, int v) {
  if (h->cfg.ma_kernel > 0) return v == 1 || v == 2;
  if (comp_on(h)) return v == 1 || v == 2 || v == 5 || (v == 6 && h->cfg.seg_len == 24);
  return v == 1 || v == 2 || v == 5 || (v == 6 && h->cfg.seg_len == 24);
}
const char* kWideningMsg =
    "metric_variant bit 1 / instance_norm need tc_quad, mma_f16x3 (N <= 32), "
    "flash_f16x3 (16 < N <= 512, S <= 96, M <= 32) or long_f32 (N <= 512); metric_variant "
    "bit 2 needs tc_quad (S = 24), mma_f16x3 (N <= 32, M <= 32, S <= 128), flash_f16x3 or "
    "long_f32; ma_kernel "
    "needs mma_f16x3 (N <= 32, M <= 32, S <= 128) or long_f32 (any N <= 512)";
// The kernels that shift the seasonal logits by a KNOWN row bound instead of searching the
// row maximum (small_f32, mma_f16x3, flash_f16x3: f_i = nu_i / sqrt(nu_i^2 + eps_s) >= rho_ij;
// DESIGN.md §3) keep the largest term of a row >= 2^(-ks/4), a normal float for
// ks = log2(e) / tau_s <= 4 x 115, i.e. tau_s >= 1/320.  Below that the row-max-searching
// FP32 kernels run (warp_f32, long_f32); tc_quad / tc_pipe (shift 1) need tau_s >= 1/80.
constexpr float kTauKnownMax = 1.0f / 320.0f;
bool known_max_ok(const prnet_handle* h) { return h->cfg.tau_seasonal >= kTauKnownMax; }
// 8 = tc_long (32 < N <= 512, S in {12, 24, 48, 96}, M <= 64, plain reading, tau_s >= 1/16:
// 128-row query tiles on tcgen05 / TMEM, key tiles of 64, known seasonal row bound f_i).  Its
// unnormalised E = 2^((rho - f_i) ks) is the P-MMA's fp16 hi/lo operand; a row whose true
// maximum f_i^2 sits below the bound (nu_i^2 not >> eps_s: f_i - f_i^2 up to 1/4) keeps its
// largest term >= 2^(-ks/4) >= 2^-5.8 only for tau_s >= 1/16 (below, fp16 subnormals lose the
// row: measured 275x the tolerance at tau_s = 0.01 on near-constant segments, DESIGN.md R-tcl)
constexpr float kTauTcl = 1.0f / 16.0f;
bool tcl_applicable(const prnet_handle* h) {
  return h->N > 32 && h->N <= 512 && h->M <= 64 && prnet::tcl_supported_s(h->cfg.seg_len) &&
         h->cfg.tau_seasonal >= kTauTcl;
}
// 9 = group_f32 (N <= 16, S <= 32: lanes over (series, segment), FP32; plain reading,
// tau_s >= 1/80 for its symmetric seasonal shift 1, as tc_quad)
bool grp_applicable(const prnet_handle* h) {
  return h->N <= 16 && h->cfg.seg_len <= 32 && h->cfg.tau_seasonal >= 0.0125f;
}
// 7 = small_f32 (N <= 16, S <= 128, M <= 32: lanes over time, FP32)
bool small_applicable(const prnet_handle* h) {
  return h->N <= 16 && h->cfg.seg_len <= 128 && h->M <= 32;
}
int pick_variant(const prnet_handle* h) {
  if (h->forced_variant >= 0) return h->forced_variant;
  // seasonal temperatures below the known-maximum kernels' domain: row-max search (FP32)
  if (!known_max_ok(h)) return (h->N <= 32 && !widening_on(h)) ? 0 : 1;
  if (widening_on(h)) {
    if (comp_on(h)) {
      // component values at S = 24 (no decomposition): tc_quad's COMP instantiation
      if (h->cfg.ma_kernel == 0 && tcq_wide_applicable(h) && h->N > 8) return 6;
      if (h->N <= 32 && h->M <= 32 && h->cfg.seg_len <= 128) return 2;
      if (h->cfg.ma_kernel == 0 && flash_applicable(h)) return 5;
      return 1;   // long_f32 (any S, N <= 512)
    }
    // (widened, the generic mma_f16x3 path is slower than tc_quad's WIDE instantiation from
    // N = 14 on: stress L336/S24 0.278 vs 0.259 ms; equal at N = 8)
    if (tcq_wide_applicable(h) && h->N > 8) return 6;
    if (h->N <= 32 && h->M <= 32 && h->cfg.seg_len <= 128) return 2;
    if (flash_applicable(h)) return 5;
    return 1;   // long_f32: any S and M (N <= 512), e.g. N <= 32 with S > 128
  }
  // measured on B200 (profiles/README.md): small_f32 is the fastest N <= 8 path (stress
  // sweep 2-9x over tc_quad / mma_f16x3) and the fastest N <= 16 path for S > 64 (2.3x);
  // tc_quad the fastest S = 24 path for N > 16 (Traffic 5.4 ms vs 6.6 ms for mma_f16x3; its
  // MMA tiles pad N to 32, so mma_f16x3 wins at N = 14: 0.166 vs 0.255 ms); mma_f16x3 the
  // fastest other N <= 32 path
  // group_f32 (lanes over (series, segment)), measured on B200 (profiles/README.md, round 2):
  // stress L96/S12 0.056 vs 0.142 ms (small_f32), L96/S24 0.038 vs 0.081, L192/S12 (N = 16)
  // 0.137 vs 0.197 (mma_f16x3), L96/S12/H720 0.210 vs 0.315 (tc_quad M <= 64); mma_f16x3 stays
  // ahead at L336/S24 (N = 14: 0.159 vs 0.170)
  if (!widening_on(h) && grp_applicable(h) &&
      (h->N <= 8 || h->cfg.seg_len <= 16 || h->M > 32))
    return 9;
  if (small_applicable(h) && (h->N <= 8 || h->cfg.seg_len > 64)) return 7;
  // tc_quad for S != 24 (fwd_tcg.cu), measured on B200 (profiles/README.md, round 2): stress
  // L336/S12 (N = 28) 0.230 vs 0.353 ms (mma_f16x3), L1440/S48 0.403 vs 0.980, L2880/S96 0.747
  // vs 2.444, L720/S48 (N = 15) 0.372 vs 0.434; mma_f16x3 stays ahead at L192/S12 (N = 16)
  if (tcq_applicable(h) &&
      (h->N > 16 || (h->N > 8 && h->cfg.seg_len == 48) || h->M > 32))   // (M > 32: else FP32)
    return 6;
  if (h->N <= 32 && h->M <= 32 && h->cfg.seg_len <= 128) return 2;
  // tc_long (tcgen05) against flash_f16x3 (mma.sync), measured on B200 (profiles/README.md,
  // round 2; S <= 24 runs two 8-softmax-warp CTAs per SM): L5760/S12 (N = 480) 25.3 vs 27.4 ms,
  // L2880/S12 7.61 vs 8.13, L1440/S12 3.22 vs 3.41, L5760/S24 11.95 vs 12.17, L5760/S96 10.5 vs
  // 11.9, L5760/S48 9.99 vs 11.6; flash stays ahead at N = 60 (S <= 48), L2880/S24 (N = 120)
  // and for S = 24 with a long head (L5760/S24/H720, M = 30: 13.4 vs 18.2 ms)
  // (last round-2 session, after the flash descriptor-phase changes: L5760/S96 (N = 60) flash 8.38
  // vs tc_long 9.72 ms; L5760/S48 (N = 120) flash 9.27 vs 9.45; L5760/S24 (N = 240) tc_long 11.15
  // vs 11.28: S >= 48 takes tc_long from N = 200 on, the S = 24 crossover)
  if (tcl_applicable(h) &&
      (!flash_applicable(h) || (h->cfg.seg_len >= 48 && h->N >= 200) ||
       (h->M <= 8 && ((h->cfg.seg_len == 12 && h->N >= 100) ||
                      (h->cfg.seg_len == 24 && h->N >= 200)))))
    return 8;   // (M > 32: the only tensor-core kernel for N > 32)
  if (h->N > 32 && flash_applicable(h)) return 5;
  return h->N <= 32 ? 0 : 1;
}

// Enqueue the forward for B windows (pointers already validated).
prnet_status enqueue_forward(prnet_handle* h, const float* x, int64_t B, float* y, float* a_s,
                             float* a_t, cudaStream_t st, int64_t slide_T = 0,
                             const float* slide_end = nullptr) {
  prnet::FwdArgs a = make_args(h, x, B, y);
  if (slide_T > 0) {  // sliding windows of a [C][T] series: window b starts at x + b
    a.xsb = 1;
    a.xsc = slide_T;
    a.x_vec = 0;
    a.x_end = slide_end;
  }
  a.a_s_dbg = a_s;
  a.a_t_dbg = a_t;
  cudaError_t e;
  int v = pick_variant(h);
  if (v < 0 || (widening_on(h) && !variant_supports_widening(h, v)))
    return fail(h, PRNET_ERR_UNSUPPORTED, kWideningMsg);
  if (a_s != nullptr) {
    // prnet_debug_attention: the dump is written by warp_f32 (the plain reading and the
    // level-only trend), mma_f16x3, long_f32 (every flag) and tc_quad (detrend /
    // instance_norm), each from the values its own fold consumes; small_f32 maps to
    // mma_f16x3 (same domain, every flag), flash_f16x3 to long_f32 (every flag and N)
    if (v == 7 || v == 9) v = h->M <= 32 ? 2 : 0;
    if (v == 5 || v == 8) v = 1;
    if (v == 0 && widening_on(h)) v = 1;
  }
  static const int wpc_env = [] {  // tuning knob: windows per CTA (0 = plan default)
    const char* e = getenv("PRNET_WINDOWS_PER_CTA");
    return e ? atoi(e) : 0;
  }();
  if (v == 9) {
    prnet::GrpPlan p;
    if (!prnet::plan_grp_kernel(a, h->max_smem_optin, &p))
      return fail(h, PRNET_ERR_UNSUPPORTED, "shape not supported by the group_f32 kernel");
    if (wpc_env > 0) p.wins_per_cta = wpc_env;
    e = prnet::launch_grp_kernel(a, p, st);
  } else if (v == 8) {
    prnet::TclPlan p;
    if (!prnet::plan_tcl_kernel(a, h->max_smem_optin, h->sm_count, &p))
      return fail(h, PRNET_ERR_UNSUPPORTED, "shape not supported by the tc_long kernel");
    e = prnet::launch_tcl_kernel(a, p, st);
  } else if (v == 7) {
    prnet::SmallPlan p;
    if (!prnet::plan_small_kernel(a, h->max_smem_optin, &p))
      return fail(h, PRNET_ERR_UNSUPPORTED, "shape not supported by the small_f32 kernel");
    if (wpc_env > 0) p.wins_per_cta = wpc_env;
    e = prnet::launch_small_kernel(a, p, st);
  } else if (v == 6 && h->cfg.seg_len == 24) {
    prnet::TcqPlan p;
    if (!prnet::plan_tcq_kernel(a, h->max_smem_optin, h->sm_count, &p))
      return fail(h, PRNET_ERR_UNSUPPORTED, "shape not supported by the tc_quad kernel");
    if (wpc_env > 0) {
      p.wins_per_group = (wpc_env + 3) & ~3;
      p.ctas_per_channel = 0;
    }
    e = prnet::launch_tcq_kernel(a, p, st);
  } else if (v == 6) {
    prnet::TcqPlan p;
    if (!prnet::plan_tcg_kernel(a, h->max_smem_optin, h->sm_count, &p))
      return fail(h, PRNET_ERR_UNSUPPORTED, "shape not supported by the tc_quad kernel");
    if (wpc_env > 0) {
      p.wins_per_group = (wpc_env + 3) & ~3;
      p.ctas_per_channel = 0;
    }
    e = prnet::launch_tcg_kernel(a, p, st);
  } else if (v == 5) {
    prnet::FlashPlan p;
    if (!prnet::plan_flash_kernel(a, h->max_smem_optin, &p))
      return fail(h, PRNET_ERR_UNSUPPORTED, "shape not supported by the flash kernel");
    e = prnet::launch_flash_kernel(a, p, st);
  } else if (v == 2) {
    prnet::MmaPlan p;
    if (!prnet::plan_mma_kernel(a, h->max_smem_optin, &p))
      return fail(h, PRNET_ERR_UNSUPPORTED, "shape not supported by the tensor-core kernel");
    if (wpc_env > 0) p.wins_per_cta = wpc_env;
    e = prnet::launch_mma_kernel(a, p, st);
  } else if (v == 0) {
    prnet::WarpPlan p;
    if (!prnet::plan_warp_kernel(a, h->max_smem_optin, &p))
      return fail(h, PRNET_ERR_UNSUPPORTED, "shape exceeds the N<=32 kernel's shared memory");
    e = prnet::launch_warp_kernel(a, p, st);
  } else {
    prnet::LongPlan p;
    if (!prnet::plan_long_kernel(a, h->max_smem_optin, h->sm_count, &p))
      return fail(h, PRNET_ERR_UNSUPPORTED, "shape exceeds the long-N kernel's limits");
    e = prnet::launch_long_kernel(a, p, st);
  }
  if (e != cudaSuccess) return cuda_fail(h, e, "forward launch");
  return PRNET_OK;
}

// The host-buffer runtime's staging rings (x: [chunk][C][L], y: [chunk][C][H], kStages
// each) and streams; x staging only when need_x (prnet_forward_host).
prnet_status ensure_staging(prnet_handle* h, int64_t chunk, bool need_x) {
  const int64_t C = h->cfg.channels, L = h->cfg.lookback, H = h->cfg.horizon;
  cudaError_t e;
  if (need_x && chunk > h->stage_windows) {
    for (int k = 0; k < prnet_handle::kStages; k++) {
      cudaFree(h->d_xstage[k]);
      h->d_xstage[k] = nullptr;
    }
    h->stage_windows = 0;
    for (int k = 0; k < prnet_handle::kStages; k++)
      if ((e = cudaMalloc(&h->d_xstage[k], chunk * C * L * 4)) != cudaSuccess)
        return cuda_fail(h, e, "cudaMalloc(x staging)");
    h->stage_windows = chunk;
  }
  if (chunk > h->ystage_windows) {
    for (int k = 0; k < prnet_handle::kStages; k++) {
      cudaFree(h->d_ystage[k]);
      h->d_ystage[k] = nullptr;
    }
    h->ystage_windows = 0;
    for (int k = 0; k < prnet_handle::kStages; k++)
      if ((e = cudaMalloc(&h->d_ystage[k], chunk * C * H * 4)) != cudaSuccess)
        return cuda_fail(h, e, "cudaMalloc(y staging)");
    h->ystage_windows = chunk;
  }
  for (int k = 0; k < prnet_handle::kStages; k++) {
    if (!h->streams[k] &&
        (e = cudaStreamCreateWithFlags(&h->streams[k], cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(h, e, "cudaStreamCreate");
  }
  return PRNET_OK;
}

prnet_status validate_forward(prnet_handle* h, const float* x, int64_t B, const float* y,
                              bool device_ptrs) {
  if (!h) return fail(nullptr, PRNET_ERR_BAD_STATE, "NULL handle");
  if (!h->loaded) return fail(h, PRNET_ERR_BAD_STATE, "forward before prnet_load_params");
  if (B < 0) return fail(h, PRNET_ERR_INVALID_ARG, "batch < 0");
  if (B == 0) return PRNET_OK;
  if (!x || !y) return fail(h, PRNET_ERR_INVALID_ARG, "NULL x or y with batch > 0");
  const int64_t C = h->cfg.channels, L = h->cfg.lookback, H = h->cfg.horizon;
  if (B > INT64_MAX / (C * (L > H ? L : H)) / 4)
    return fail(h, PRNET_ERR_INVALID_ARG, "batch * C * L overflows");
  if (device_ptrs) {
    if (((uintptr_t)x & 15) || ((uintptr_t)y & 15))
      return fail(h, PRNET_ERR_UNSUPPORTED, "x and y must be 16-byte aligned");
    if (overlaps(x, (size_t)(B * C * L * 4), y, (size_t)(B * C * H * 4)))
      return fail(h, PRNET_ERR_UNSUPPORTED, "x and y overlap");
    prnet_status s = check_dev_ptr(h, x, "x");
    if (s != PRNET_OK) return s;
    s = check_dev_ptr(h, y, "y");
    if (s != PRNET_OK) return s;
  } else if (overlaps(x, (size_t)(B * C * L * 4), y, (size_t)(B * C * H * 4))) {
    return fail(h, PRNET_ERR_UNSUPPORTED, "x and y overlap");
  }
  return PRNET_OK;
}

}  // namespace

extern "C" {

prnet_status prnet_create(const prnet_config* cfg, prnet_handle** out) {
  if (out) *out = nullptr;
  if (!cfg || !out) return fail(nullptr, PRNET_ERR_INVALID_ARG, "NULL cfg or out");
  if (cfg->abi_version < 1 || cfg->abi_version > PRNET_ABI_VERSION)
    return fail(nullptr, PRNET_ERR_INVALID_ARG, "abi_version must be 1, 2 or 3");
  // a v1 caller's struct ends at `device`, a v2 caller's at `instance_norm`: copy only what
  // the caller owns
  prnet_config c2{};
  if (cfg->abi_version == 1)
    std::memcpy(&c2, cfg, offsetof(prnet_config, instance_norm));
  else if (cfg->abi_version == 2)
    std::memcpy(&c2, cfg, offsetof(prnet_config, ma_kernel));
  else
    c2 = *cfg;
  c2.abi_version = PRNET_ABI_VERSION;
  cfg = &c2;
  if (cfg->channels < 1 || cfg->seg_len < 2 || cfg->lookback < cfg->seg_len || cfg->horizon < 1)
    return fail(nullptr, PRNET_ERR_INVALID_ARG, "need C >= 1, S >= 2, L >= S, H >= 1");
  if (!(cfg->tau_seasonal > 0.f) || !std::isfinite(cfg->tau_seasonal) ||
      !(cfg->tau_trend > 0.f) || !std::isfinite(cfg->tau_trend))
    return fail(nullptr, PRNET_ERR_INVALID_ARG, "temperatures must be finite and > 0");
  if (cfg->metric_variant < 0 || cfg->metric_variant > 7)
    return fail(nullptr, PRNET_ERR_INVALID_ARG,
                "metric_variant must be in [0, 7] (bit 0 level trend, bit 1 detrended seasonal, "
                "bit 2 component values)");
  if (cfg->instance_norm != 0 && cfg->instance_norm != 1)
    return fail(nullptr, PRNET_ERR_INVALID_ARG, "instance_norm must be 0 or 1");
  if (cfg->ma_kernel < 0 || cfg->ma_kernel > 4095 ||
      (cfg->ma_kernel > 0 && (cfg->ma_kernel & 1) == 0))
    return fail(nullptr, PRNET_ERR_INVALID_ARG, "ma_kernel must be 0 or odd in [1, 4095]");
  if (cfg->channels > 65535)
    return fail(nullptr, PRNET_ERR_UNSUPPORTED, "C > 65535 not supported");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || cfg->device < 0 || cfg->device >= ndev) {
    cudaGetLastError();
    return fail(nullptr, PRNET_ERR_UNSUPPORTED, "no such CUDA device");
  }
  cudaDeviceProp prop;
  if ((e = cudaGetDeviceProperties(&prop, cfg->device)) != cudaSuccess)
    return cuda_fail(nullptr, e, "cudaGetDeviceProperties");
  if (prop.major != 10)
    return fail(nullptr, PRNET_ERR_UNSUPPORTED,
                "device is not compute capability 10.x (this library is built for sm_100a)");
  prnet_handle* h = new (std::nothrow) prnet_handle();
  if (!h) return fail(nullptr, PRNET_ERR_OOM, "host allocation failed");
  h->cfg = *cfg;
  h->N = cfg->lookback / cfg->seg_len;
  h->r = cfg->lookback - h->N * cfg->seg_len;
  h->M = (cfg->horizon + cfg->seg_len - 1) / cfg->seg_len;
  h->Cw = cfg->head_per_channel ? cfg->channels : 1;
  h->sm_count = prop.multiProcessorCount;
  h->max_smem_optin = (int)prop.sharedMemPerBlockOptin;
  if (h->N > 512 || cfg->seg_len > 4096) {
    delete h;
    return fail(nullptr, PRNET_ERR_UNSUPPORTED, "N > 512 segments not supported");
  }
  DeviceGuard g(cfg->device);
  const size_t nw = (size_t)h->Cw * h->M * h->N, nb = (size_t)h->Cw * cfg->horizon;
  if ((e = cudaMalloc(&h->d_ws, nw * 4)) != cudaSuccess ||
      (e = cudaMalloc(&h->d_wt, nw * 4)) != cudaSuccess ||
      (e = cudaMalloc(&h->d_b, nb * 4)) != cudaSuccess ||
      (e = cudaMalloc(&h->d_err, 2 * prnet::kErrPartials * sizeof(double))) != cudaSuccess) {
    prnet_status s = cuda_fail(nullptr, e, "cudaMalloc(params)");
    prnet_destroy(h);
    return s;
  }
  *out = h;
  return PRNET_OK;
}

prnet_status prnet_load_params(prnet_handle* h, const float* w_seasonal, const float* w_trend,
                               const float* bias, int64_t n_w, int64_t n_b) {
  if (!h) return fail(nullptr, PRNET_ERR_BAD_STATE, "NULL handle");
  const int64_t want_w = (int64_t)h->Cw * h->M * h->N, want_b = (int64_t)h->Cw * h->cfg.horizon;
  if (!w_seasonal || !w_trend || !bias) return fail(h, PRNET_ERR_INVALID_ARG, "NULL parameter");
  if (n_w != want_w || n_b != want_b)
    return fail(h, PRNET_ERR_INVALID_ARG,
                "parameter counts: want n_w=" + std::to_string(want_w) +
                    " n_b=" + std::to_string(want_b));
  DeviceGuard g(h->cfg.device);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(h, e, "cudaDeviceSynchronize");
  if ((e = cudaMemcpy(h->d_ws, w_seasonal, want_w * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(h->d_wt, w_trend, want_w * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(h->d_b, bias, want_b * 4, cudaMemcpyHostToDevice)) != cudaSuccess)
    return cuda_fail(h, e, "cudaMemcpy(params)");
  if (h->N <= 32 && h->M <= 32) {  // pre-pack the head for the tensor-core variant
    const int bytes = prnet::mma_wpack_bytes(h->N, h->M);
    std::vector<unsigned char> pack((size_t)h->Cw * bytes);
    std::vector<float> inv(h->Cw);
    prnet::pack_mma_head(w_seasonal, w_trend, h->Cw, h->M, h->N, pack.data(), inv.data());
    if (!h->d_wpack) {
      if ((e = cudaMalloc(&h->d_wpack, pack.size())) != cudaSuccess ||
          (e = cudaMalloc(&h->d_invsw, inv.size() * 4)) != cudaSuccess)
        return cuda_fail(h, e, "cudaMalloc(packed head)");
    }
    if ((e = cudaMemcpy(h->d_wpack, pack.data(), pack.size(), cudaMemcpyHostToDevice)) !=
            cudaSuccess ||
        (e = cudaMemcpy(h->d_invsw, inv.data(), inv.size() * 4, cudaMemcpyHostToDevice)) !=
            cudaSuccess)
      return cuda_fail(h, e, "cudaMemcpy(packed head)");
  }
  if (flash_applicable(h) || tcl_applicable(h)) {  // head for the key-streaming kernels
    const int bytes = prnet::flash_wpack_bytes(h->N, h->M);
    std::vector<unsigned char> pack((size_t)h->Cw * bytes);
    std::vector<float> inv(h->Cw);
    prnet::pack_flash_head(w_seasonal, w_trend, h->Cw, h->M, h->N, pack.data(), inv.data());
    if (!h->d_wpack_fl && ((e = cudaMalloc(&h->d_wpack_fl, pack.size())) != cudaSuccess ||
                           (e = cudaMalloc(&h->d_invsw_fl, inv.size() * 4)) != cudaSuccess))
      return cuda_fail(h, e, "cudaMalloc(flash head)");
    if ((e = cudaMemcpy(h->d_wpack_fl, pack.data(), pack.size(), cudaMemcpyHostToDevice)) !=
            cudaSuccess ||
        (e = cudaMemcpy(h->d_invsw_fl, inv.data(), inv.size() * 4, cudaMemcpyHostToDevice)) !=
            cudaSuccess)
      return cuda_fail(h, e, "cudaMemcpy(flash head)");
  }
  if (tc_head_shape(h)) {  // the same head as the tcgen05 B operand (K-major core matrices)
    const int bytes = prnet::tc_wpack_bytes(h->M);
    std::vector<unsigned char> pack((size_t)h->Cw * bytes);
    std::vector<float> inv(h->Cw);
    prnet::pack_tc_head(w_seasonal, w_trend, h->Cw, h->M, h->N, pack.data(), inv.data());
    if (!h->d_wpack_tc && (e = cudaMalloc(&h->d_wpack_tc, pack.size())) != cudaSuccess)
      return cuda_fail(h, e, "cudaMalloc(tc head)");
    if ((e = cudaMemcpy(h->d_wpack_tc, pack.data(), pack.size(), cudaMemcpyHostToDevice)) !=
        cudaSuccess)
      return cuda_fail(h, e, "cudaMemcpy(tc head)");
    // 1 / sw (the same power-of-two scale as the mma pack's, which M > 32 handles do not build)
    if (!h->d_invsw && (e = cudaMalloc(&h->d_invsw, inv.size() * 4)) != cudaSuccess)
      return cuda_fail(h, e, "cudaMalloc(tc head scale)");
    if ((e = cudaMemcpy(h->d_invsw, inv.data(), inv.size() * 4, cudaMemcpyHostToDevice)) !=
        cudaSuccess)
      return cuda_fail(h, e, "cudaMemcpy(tc head scale)");
  }
  h->loaded = true;
  return PRNET_OK;
}

prnet_status prnet_forward(prnet_handle* h, const float* x, int64_t batch, float* y,
                           void* cuda_stream) {
  prnet_status s = validate_forward(h, x, batch, y, true);
  if (s != PRNET_OK || batch == 0) return s;
  DeviceGuard g(h->cfg.device);
  return enqueue_forward(h, x, batch, y, nullptr, nullptr, (cudaStream_t)cuda_stream);
}

prnet_status prnet_set_host_chunk(prnet_handle* h, int64_t windows_per_chunk) {
  if (!h) return fail(nullptr, PRNET_ERR_BAD_STATE, "NULL handle");
  if (windows_per_chunk < 1) return fail(h, PRNET_ERR_INVALID_ARG, "windows_per_chunk < 1");
  h->host_chunk = windows_per_chunk;
  return PRNET_OK;
}

prnet_status prnet_forward_host(prnet_handle* h, const float* x_host, int64_t batch,
                                float* y_host) {
  prnet_status s = validate_forward(h, x_host, batch, y_host, false);
  if (s != PRNET_OK || batch == 0) return s;
  DeviceGuard g(h->cfg.device);
  const int64_t C = h->cfg.channels, L = h->cfg.lookback, H = h->cfg.horizon;
  int64_t chunk = h->host_chunk;
  if (chunk <= 0) {
    chunk = (256ll << 20) / (C * L * 4);
    if (chunk < 1) chunk = 1;
  }
  if (chunk > batch) chunk = batch;
  cudaError_t e;
  if ((s = ensure_staging(h, chunk, true)) != PRNET_OK) return s;
  // Chunk k goes to stage k % 3 on stream k % 3: H2D -> kernel -> D2H in stream
  // order, so the copy engines overlap chunk k+1's upload, chunk k's kernel and
  // chunk k-1's download across the three streams.
  int64_t k = 0;
  for (int64_t b0 = 0; b0 < batch; b0 += chunk, k++) {
    const int64_t nb = (batch - b0) < chunk ? (batch - b0) : chunk;
    const int st = (int)(k % prnet_handle::kStages);
    cudaStream_t stream = h->streams[st];
    if ((e = cudaMemcpyAsync(h->d_xstage[st], x_host + b0 * C * L, nb * C * L * 4,
                             cudaMemcpyHostToDevice, stream)) != cudaSuccess)
      return cuda_fail(h, e, "cudaMemcpyAsync(H2D)");
    s = enqueue_forward(h, h->d_xstage[st], nb, h->d_ystage[st], nullptr, nullptr, stream);
    if (s != PRNET_OK) return s;
    if ((e = cudaMemcpyAsync(y_host + b0 * C * H, h->d_ystage[st], nb * C * H * 4,
                             cudaMemcpyDeviceToHost, stream)) != cudaSuccess)
      return cuda_fail(h, e, "cudaMemcpyAsync(D2H)");
  }
  for (int st = 0; st < prnet_handle::kStages; st++)
    if ((e = cudaStreamSynchronize(h->streams[st])) != cudaSuccess)
      return cuda_fail(h, e, "cudaStreamSynchronize");
  return PRNET_OK;
}

// ---- sliding-window input mode
static prnet_status validate_sliding(prnet_handle* h, const float* series, int64_t T, int64_t t0,
                              int64_t B, const float* y, bool device_ptrs) {
  if (!h) return fail(nullptr, PRNET_ERR_BAD_STATE, "NULL handle");
  if (!h->loaded) return fail(h, PRNET_ERR_BAD_STATE, "forward before prnet_load_params");
  if (B < 0) return fail(h, PRNET_ERR_INVALID_ARG, "batch < 0");
  if (B == 0) return PRNET_OK;
  if (!series || !y) return fail(h, PRNET_ERR_INVALID_ARG, "NULL series or y with batch > 0");
  const int64_t C = h->cfg.channels, L = h->cfg.lookback, H = h->cfg.horizon;
  if (t0 < 0 || T < L || B > T - L - t0 + 1)
    return fail(h, PRNET_ERR_INVALID_ARG, "need 0 <= t0 and t0 + batch - 1 + L <= T");
  if (T > INT64_MAX / C / 4 || B > INT64_MAX / (C * H) / 4)
    return fail(h, PRNET_ERR_INVALID_ARG, "size overflows");
  if (overlaps(series, (size_t)(C * T * 4), y, (size_t)(B * C * H * 4)))
    return fail(h, PRNET_ERR_UNSUPPORTED, "series and y overlap");
  if (device_ptrs) {
    if (((uintptr_t)series & 15) || ((uintptr_t)y & 15))
      return fail(h, PRNET_ERR_UNSUPPORTED, "series and y must be 16-byte aligned");
    prnet_status s = check_dev_ptr(h, series, "series");
    if (s != PRNET_OK) return s;
    s = check_dev_ptr(h, y, "y");
    if (s != PRNET_OK) return s;
  }
  return PRNET_OK;
}

prnet_status prnet_forward_sliding(prnet_handle* h, const float* series, int64_t T, int64_t t0,
                                   int64_t batch, float* y, void* cuda_stream) {
  prnet_status s = validate_sliding(h, series, T, t0, batch, y, true);
  if (s != PRNET_OK || batch == 0) return s;
  DeviceGuard g(h->cfg.device);
  return enqueue_forward(h, series + t0, batch, y, nullptr, nullptr, (cudaStream_t)cuda_stream,
                         T, series + h->cfg.channels * T);
}

prnet_status prnet_forward_sliding_host(prnet_handle* h, const float* series, int64_t T,
                                        int64_t t0, int64_t batch, float* y_host) {
  prnet_status s = validate_sliding(h, series, T, t0, batch, y_host, false);
  if (s != PRNET_OK || batch == 0) return s;
  DeviceGuard g(h->cfg.device);
  const int64_t C = h->cfg.channels, L = h->cfg.lookback, H = h->cfg.horizon;
  const int64_t span = batch - 1 + L;          // the time steps every window touches
  const int64_t Tp = (span + 3) & ~int64_t(3);  // 16-byte pitch of the device copy
  cudaError_t e;
  if (C * Tp > h->series_floats) {
    cudaFree(h->d_series);
    h->d_series = nullptr;
    h->series_floats = 0;
    if ((e = cudaMalloc(&h->d_series, C * Tp * 4)) != cudaSuccess)
      return cuda_fail(h, e, "cudaMalloc(series)");
    h->series_floats = C * Tp;
  }
  int64_t chunk = h->host_chunk;
  if (chunk <= 0) {
    chunk = (128ll << 20) / (C * H * 4);
    if (chunk < 1) chunk = 1;
  }
  if (chunk > batch) chunk = batch;
  // only the output staging ring: the windows are read from the uploaded series span
  if ((s = ensure_staging(h, chunk, false)) != PRNET_OK) return s;
  // the series span goes up once (C rows of `span` floats, pitched); windows are then
  // forecast in chunks on three streams so chunk k's D2H overlaps chunk k+1's kernel
  if ((e = cudaMemcpy2DAsync(h->d_series, Tp * 4, series + t0, T * 4, span * 4, C,
                             cudaMemcpyHostToDevice, h->streams[0])) != cudaSuccess)
    return cuda_fail(h, e, "cudaMemcpy2DAsync(series)");
  cudaEvent_t up;
  if ((e = cudaEventCreateWithFlags(&up, cudaEventDisableTiming)) != cudaSuccess)
    return cuda_fail(h, e, "cudaEventCreate");
  cudaEventRecord(up, h->streams[0]);
  for (int k = 1; k < prnet_handle::kStages; k++) cudaStreamWaitEvent(h->streams[k], up, 0);
  cudaEventDestroy(up);
  int64_t k = 0;
  for (int64_t b0 = 0; b0 < batch; b0 += chunk, k++) {
    const int64_t nb = (batch - b0) < chunk ? (batch - b0) : chunk;
    const int st = (int)(k % prnet_handle::kStages);
    cudaStream_t stream = h->streams[st];
    s = enqueue_forward(h, h->d_series + b0, nb, h->d_ystage[st], nullptr, nullptr, stream, Tp,
                        h->d_series + C * Tp);
    if (s != PRNET_OK) return s;
    if ((e = cudaMemcpyAsync(y_host + b0 * C * H, h->d_ystage[st], nb * C * H * 4,
                             cudaMemcpyDeviceToHost, stream)) != cudaSuccess)
      return cuda_fail(h, e, "cudaMemcpyAsync(D2H)");
  }
  for (int st = 0; st < prnet_handle::kStages; st++)
    if ((e = cudaStreamSynchronize(h->streams[st])) != cudaSuccess)
      return cuda_fail(h, e, "cudaStreamSynchronize");
  return PRNET_OK;
}

void prnet_destroy(prnet_handle* h) {
  if (!h) return;
  {
    DeviceGuard g(h->cfg.device);
    cudaFree(h->d_series);
    cudaFree(h->d_bwd);
    cudaFree(h->d_ws);
    cudaFree(h->d_wt);
    cudaFree(h->d_b);
    cudaFree(h->d_err);
    cudaFree(h->d_wpack);
    cudaFree(h->d_invsw);
    cudaFree(h->d_wpack_tc);
    cudaFree(h->d_wpack_fl);
    cudaFree(h->d_invsw_fl);
    for (int k = 0; k < prnet_handle::kStages; k++) {
      cudaFree(h->d_xstage[k]);
      cudaFree(h->d_ystage[k]);
      if (h->streams[k]) cudaStreamDestroy(h->streams[k]);
    }
  }
  delete h;
}

const char* prnet_last_error(const prnet_handle* h) {
  if (!h) return g_create_error.c_str();
  // a per-thread copy: another thread may overwrite h->err while the caller reads it
  thread_local std::string copy;
  {
    std::lock_guard<std::mutex> lk(h->err_mu);
    copy = h->err;
  }
  return copy.c_str();
}

prnet_status prnet_get_dims(const prnet_handle* h, int32_t* N, int32_t* M, int32_t* r) {
  if (!h) return fail(nullptr, PRNET_ERR_BAD_STATE, "NULL handle");
  if (N) *N = h->N;
  if (M) *M = h->M;
  if (r) *r = h->r;
  return PRNET_OK;
}

prnet_status prnet_debug_segments(prnet_handle* h, const float* x, int64_t batch, float* seg,
                                  void* cuda_stream) {
  if (!h) return fail(nullptr, PRNET_ERR_BAD_STATE, "NULL handle");
  if (batch < 0) return fail(h, PRNET_ERR_INVALID_ARG, "batch < 0");
  if (batch == 0) return PRNET_OK;
  if (!x || !seg) return fail(h, PRNET_ERR_INVALID_ARG, "NULL pointer");
  prnet_status s = check_dev_ptr(h, x, "x");
  if (s == PRNET_OK) s = check_dev_ptr(h, seg, "seg");
  if (s != PRNET_OK) return s;
  DeviceGuard g(h->cfg.device);
  cudaError_t e = prnet::launch_gather_segments(x, batch, h->cfg.channels, h->cfg.lookback,
                                                h->cfg.seg_len, h->N, h->r, seg,
                                                (cudaStream_t)cuda_stream);
  return e == cudaSuccess ? PRNET_OK : cuda_fail(h, e, "gather_segments launch");
}

prnet_status prnet_debug_attention(prnet_handle* h, const float* x, int64_t batch, float* a_s,
                                   float* a_t, void* cuda_stream) {
  if (!h) return fail(nullptr, PRNET_ERR_BAD_STATE, "NULL handle");
  if (!a_s || !a_t) return fail(h, PRNET_ERR_INVALID_ARG, "NULL attention buffer");
  const int64_t C = h->cfg.channels, H = h->cfg.horizon;
  prnet_status s = validate_forward(h, x, batch, a_s, true);  // x checks (a_s as dummy y)
  if (s != PRNET_OK || batch == 0) return s;
  s = check_dev_ptr(h, a_t, "a_t");
  if (s != PRNET_OK) return s;
  DeviceGuard g(h->cfg.device);
  // the forward's own y goes to a scratch buffer
  float* y = nullptr;
  cudaError_t e = cudaMallocAsync(&y, batch * C * H * 4, (cudaStream_t)cuda_stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "cudaMallocAsync(scratch y)");
  s = enqueue_forward(h, x, batch, y, a_s, a_t, (cudaStream_t)cuda_stream);
  cudaFreeAsync(y, (cudaStream_t)cuda_stream);
  return s;
}

prnet_status prnet_error_sums(prnet_handle* h, const float* y, const float* target,
                              int64_t batch, double* out3, void* cuda_stream) {
  if (!h) return fail(nullptr, PRNET_ERR_BAD_STATE, "NULL handle");
  if (batch < 0 || !y || !target || !out3)
    return fail(h, PRNET_ERR_INVALID_ARG, "NULL pointer or batch < 0");
  prnet_status s = check_dev_ptr(h, y, "y");
  if (s == PRNET_OK) s = check_dev_ptr(h, target, "target");
  if (s == PRNET_OK) s = check_dev_ptr(h, out3, "out3");
  if (s != PRNET_OK) return s;
  DeviceGuard g(h->cfg.device);
  const int64_t n = batch * h->cfg.channels * h->cfg.horizon;
  cudaError_t e = prnet::launch_error_sums(y, target, n, h->d_err, out3, (cudaStream_t)cuda_stream);
  return e == cudaSuccess ? PRNET_OK : cuda_fail(h, e, "error_sums launch");
}

prnet_status prnet_backward_head(prnet_handle* h, const float* x, int64_t batch,
                                 const float* dy, float* dws, float* dwt, float* db,
                                 void* cuda_stream) {
  if (!h) return fail(nullptr, PRNET_ERR_BAD_STATE, "NULL handle");
  if (batch < 0) return fail(h, PRNET_ERR_INVALID_ARG, "batch < 0");
  if (!dws || !dwt || !db || (batch > 0 && (!x || !dy)))
    return fail(h, PRNET_ERR_INVALID_ARG, "NULL pointer");
  if ((h->cfg.metric_variant & 4) != 0 || h->cfg.ma_kernel > 0)
    return fail(h, PRNET_ERR_UNSUPPORTED,
                "backward_head: component values and the decomposition are forward-only");
  prnet_status s = PRNET_OK;
  if (batch > 0) {
    s = check_dev_ptr(h, x, "x");
    if (s == PRNET_OK) s = check_dev_ptr(h, dy, "dy");
  }
  if (s == PRNET_OK) s = check_dev_ptr(h, dws, "dws");
  if (s == PRNET_OK) s = check_dev_ptr(h, dwt, "dwt");
  if (s == PRNET_OK) s = check_dev_ptr(h, db, "db");
  if (s != PRNET_OK) return s;
  DeviceGuard g(h->cfg.device);
  prnet::FwdArgs a = make_args(h, x, batch, nullptr);
  prnet::BwdPlan p;
  if (!prnet::plan_bwd_head(a, h->max_smem_optin, &p))
    return fail(h, PRNET_ERR_UNSUPPORTED, "backward_head needs N <= 512, M <= 32 (and the "
                                          "long-lookback rows within shared memory)");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int64_t need = (int64_t)h->cfg.channels * p.nblk * p.elems;
  if (need > h->bwd_floats) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(h, e, "backward_head sync");
    cudaFree(h->d_bwd);
    h->d_bwd = nullptr;
    h->bwd_floats = 0;
    e = cudaMalloc(&h->d_bwd, (size_t)need * sizeof(float));
    if (e != cudaSuccess) return cuda_fail(h, e, "backward_head workspace");
    h->bwd_floats = need;
  }
  cudaError_t e = prnet::launch_bwd_head(a, p, dy, h->d_bwd, dws, dwt, db, h->Cw, st);
  return e == cudaSuccess ? PRNET_OK : cuda_fail(h, e, "backward_head launch");
}

prnet_status prnet_forward_bf16(prnet_handle* h, const uint16_t* x, int64_t batch, uint16_t* y,
                                void* cuda_stream) {
  if (!h) return fail(nullptr, PRNET_ERR_BAD_STATE, "NULL handle");
  if (!h->loaded) return fail(h, PRNET_ERR_BAD_STATE, "forward before prnet_load_params");
  if (batch < 0) return fail(h, PRNET_ERR_INVALID_ARG, "batch < 0");
  if (batch > 0 && (!x || !y)) return fail(h, PRNET_ERR_INVALID_ARG, "NULL pointer");
  if (!tcq_wide_applicable(h) || widening_on(h) || (h->cfg.metric_variant & 1) != 0)
    return fail(h, PRNET_ERR_UNSUPPORTED,
                "forward_bf16 runs the S = 24 tc_quad kernel: N <= 32, M <= 32, "
                "tau_seasonal >= 1/80, the base reading");
  if (batch == 0) return PRNET_OK;
  prnet_status s = check_dev_ptr(h, x, "x");
  if (s == PRNET_OK) s = check_dev_ptr(h, y, "y");
  if (s != PRNET_OK) return s;
  const int64_t C = h->cfg.channels, L = h->cfg.lookback, H = h->cfg.horizon;
  if (((uintptr_t)x & 3u) != 0 || ((uintptr_t)y & 3u) != 0)
    return fail(h, PRNET_ERR_UNSUPPORTED, "x / y not 4-byte aligned");
  if (overlaps(x, (size_t)(batch * C * L) * 2, y, (size_t)(batch * C * H) * 2))
    return fail(h, PRNET_ERR_UNSUPPORTED, "x and y overlap");
  DeviceGuard g(h->cfg.device);
  prnet::FwdArgs a = make_args(h, reinterpret_cast<const float*>(x), batch,
                               reinterpret_cast<float*>(y));
  a.io_bf16 = 1;
  // one 1-D bulk copy per series: 16-byte aligned bf16 window starts
  a.x_vec = (L % 8 == 0) && (h->r % 8 == 0) && (((uintptr_t)x & 15u) == 0);
  prnet::TcqPlan p;
  if (!prnet::plan_tcq_kernel(a, h->max_smem_optin, h->sm_count, &p))
    return fail(h, PRNET_ERR_UNSUPPORTED, "shape not supported by the tc_quad kernel");
  cudaError_t e = prnet::launch_tcq_kernel(a, p, (cudaStream_t)cuda_stream);
  return e == cudaSuccess ? PRNET_OK : cuda_fail(h, e, "forward_bf16 launch");
}

prnet_status prnet_backward(prnet_handle* h, const float* x, int64_t batch, const float* dy,
                            float* dx, float* dws, float* dwt, float* db, float* dtau,
                            void* cuda_stream) {
  if (!h) return fail(nullptr, PRNET_ERR_BAD_STATE, "NULL handle");
  if (!h->loaded) return fail(h, PRNET_ERR_BAD_STATE, "backward before prnet_load_params");
  if (batch < 0) return fail(h, PRNET_ERR_INVALID_ARG, "batch < 0");
  if (!dws || !dwt || !db || !dtau || (batch > 0 && (!x || !dy || !dx)))
    return fail(h, PRNET_ERR_INVALID_ARG, "NULL pointer");
  if ((h->cfg.metric_variant & ~1) != 0 || h->cfg.instance_norm || h->cfg.ma_kernel > 0)
    return fail(h, PRNET_ERR_UNSUPPORTED,
                "backward: the base reading only (metric_variant 0 or 1, no instance_norm, no "
                "ma_kernel)");
  prnet_status s = PRNET_OK;
  if (batch > 0) {
    s = check_dev_ptr(h, x, "x");
    if (s == PRNET_OK) s = check_dev_ptr(h, dy, "dy");
    if (s == PRNET_OK) s = check_dev_ptr(h, dx, "dx");
  }
  if (s == PRNET_OK) s = check_dev_ptr(h, dws, "dws");
  if (s == PRNET_OK) s = check_dev_ptr(h, dwt, "dwt");
  if (s == PRNET_OK) s = check_dev_ptr(h, db, "db");
  if (s == PRNET_OK) s = check_dev_ptr(h, dtau, "dtau");
  if (s != PRNET_OK) return s;
  DeviceGuard g(h->cfg.device);
  prnet::FwdArgs a = make_args(h, x, batch, nullptr);
  prnet::BwdFullPlan p;
  if (!prnet::plan_bwd_full(a, h->max_smem_optin, &p))
    return fail(h, PRNET_ERR_UNSUPPORTED, "backward needs N <= 32, M <= 32, S <= 128");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int64_t need = (int64_t)prnet::bwd_full_workspace_floats(a, p);
  if (need > h->bwd_floats) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(h, e, "backward sync");
    cudaFree(h->d_bwd);
    h->d_bwd = nullptr;
    h->bwd_floats = 0;
    e = cudaMalloc(&h->d_bwd, (size_t)need * sizeof(float));
    if (e != cudaSuccess) return cuda_fail(h, e, "backward workspace");
    h->bwd_floats = need;
  }
  cudaError_t e = prnet::launch_bwd_full(a, p, dy, dx, h->d_bwd, dws, dwt, db, dtau, h->Cw, st);
  return e == cudaSuccess ? PRNET_OK : cuda_fail(h, e, "backward launch");
}

prnet_status prnet_set_kernel_variant(prnet_handle* h, int32_t variant) {
  if (!h) return fail(nullptr, PRNET_ERR_BAD_STATE, "NULL handle");
  if (variant < -1 || variant > 9)
    return fail(h, PRNET_ERR_INVALID_ARG, "variant in {-1,...,9}");
  if (variant == 9 && !grp_applicable(h))
    return fail(h, PRNET_ERR_UNSUPPORTED,
                "group_f32 variant needs N <= 16, S <= 32, tau_seasonal >= 1/80");
  if (variant == 8 && !tcl_applicable(h))
    return fail(h, PRNET_ERR_UNSUPPORTED,
                "tc_long variant needs 32 < N <= 512, S in {12, 24, 48, 96}, M <= 64, "
                "tau_seasonal >= 1/16");
  if (variant == 3 || variant == 4)
    return fail(h, PRNET_ERR_INVALID_ARG,
                "variants 3 (tc_fold) and 4 (tc_full) are retired: 6 (tc_quad) supersedes them");
  if (variant == 7 && !small_applicable(h))
    return fail(h, PRNET_ERR_UNSUPPORTED, "small_f32 variant needs N <= 16, S <= 128, M <= 32");
  if (variant == 6 && !tcq_applicable(h))
    return fail(h, PRNET_ERR_UNSUPPORTED,
                "tc_quad variant needs S in {12, 16, 24, 32, 48, 64, 96}, N <= 32, M <= 32 (S = 24) or M <= 64, tau_seasonal >= 1/80");
  if ((variant == 2 || variant == 5 || variant == 7) && !known_max_ok(h))
    return fail(h, PRNET_ERR_UNSUPPORTED,
                "small_f32 / mma_f16x3 / flash_f16x3 need tau_seasonal >= 1/320 (known-maximum "
                "softmax shift); warp_f32 and long_f32 take any temperature");
  if (variant == 5 && !flash_applicable(h))
    return fail(h, PRNET_ERR_UNSUPPORTED, "flash variant needs 16 < N <= 512, S <= 96, M <= 32");
  if ((variant == 0 || variant == 2) && h->N > 32)
    return fail(h, PRNET_ERR_UNSUPPORTED, "variant needs N <= 32");
  if (variant == 2 && (h->M > 32 || h->cfg.seg_len > 128))
    return fail(h, PRNET_ERR_UNSUPPORTED, "tensor-core variant needs M <= 32 and S <= 128");
  if (variant >= 0 && widening_on(h) && !variant_supports_widening(h, variant))
    return fail(h, PRNET_ERR_UNSUPPORTED, kWideningMsg);
  h->forced_variant = variant;
  return PRNET_OK;
}

prnet_status prnet_forward_plan(const prnet_handle* h, int64_t batch, int32_t* kernel_launches,
                                int32_t* variant) {
  if (!h) return fail(nullptr, PRNET_ERR_BAD_STATE, "NULL handle");
  if (kernel_launches) *kernel_launches = batch > 0 ? 1 : 0;
  if (variant) *variant = pick_variant(h);
  return PRNET_OK;
}

}  // extern "C"
