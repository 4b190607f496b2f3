// fwd_warp.cu -- fused PRNet pattern-attention forward for N <= 32 segments
// per series (every configs[0..3] shape and the short-lookback stress points).
//
// One warp owns one (window, channel) series at a time; lane i owns segment
// row i.  A CTA owns one channel c and a block of windows, so the channel's
// head (W_s, W_t, b) is staged in shared memory once per CTA.  Every step of
// DESIGN.md §3 runs in this one kernel, in shared memory and registers; the
// series is read from HBM once (128-bit streaming loads) and y written once.
//
// Step map (reading of DESIGN.md §3):
//   a1 segment      xs[n][t] = x[r + n S + t]                 (Def 2, A2)
//   a2 descriptors  mu_n, z_n, nu2_n, kappa_n, sigma^2       (Def 3-5)
//   a3 seasonal     rho_ij = <z_i,z_j> / sqrt((nu2_i+e)(nu2_j+e))   (Def 6)
//   a4 trend        Dhat_ij = [dmu^2 + (S^2-1)/12 dkappa^2] / (sigma^2+e_t) (Def 7)
//   a5 softmax      A_s = softmax_j(rho/tau_s), A_t = softmax_j(-Dhat/tau_t) (Def 8)
//   a6+a7 fold      Q = W_s A_s + W_t A_t  (M x N),  Y = Q X  (M x S)   (Def 9-10,
//                   associativity: W (A X) = (W A) X)
//   a8 store        y[h] = Y[h / S][h % S] + b[h]                    (Def 11)
#include "prnet_internal.cuh"

namespace prnet {

template <int NMAX>
__global__ void __launch_bounds__(256) prnet_fwd_warp_kernel(FwdArgs a, int wins_per_cta,
                                                             int per_warp, int off_r2, int off_r3,
                                                             int shared_floats) {
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int c = blockIdx.y;
  const int cw = a.head_per_channel ? c : 0;
  const int S = a.S, N = a.N, M = a.M, H = a.H, C = a.C;
  const int SP = (S + 3) & ~3;       // padded row stride of xs (16-byte rows)
  constexpr int AP = NMAX + 1;       // odd stride: conflict-free row writes / column reads
  constexpr int QP = NMAX + 1;
  const int YP = S | 1;              // odd stride of the Y staging rows

  // ---- CTA-shared head of channel c: W_s, W_t padded to [M][NMAX] (zeros past N), b[H]
  float* wsS = smem;
  float* wtS = wsS + M * NMAX;
  float* bS = wtS + M * NMAX;
  {
    const float* gws = a.ws + (int64_t)cw * M * N;
    const float* gwt = a.wt + (int64_t)cw * M * N;
    for (int k = threadIdx.x; k < M * NMAX; k += blockDim.x) {
      int m = k / NMAX, n = k - m * NMAX;
      wsS[k] = n < N ? gws[m * N + n] : 0.f;
      wtS[k] = n < N ? gwt[m * N + n] : 0.f;
    }
    const float* gb = a.bias + (int64_t)cw * H;
    for (int k = threadIdx.x; k < H; k += blockDim.x) bS[k] = gb[k];
  }
  float* wb = smem + shared_floats + warp * per_warp;
  float* xs = wb;                 // [NMAX][SP]   natural segments (rows >= N stay 0)
  float* zt = wb + off_r2;        // [S][NMAX]    z transposed      (steps a2-a3)
  float* qs = wb + off_r2;        // [M][QP]      Q = W A           (aliases zt)
  float* as_ = wb + off_r3;       // [NMAX][AP]   A_s rows
  float* at_ = as_ + NMAX * AP;   // [NMAX][AP]   A_t rows
  float* ys = wb + off_r3;        // [M][YP]      Y staging         (aliases A)
  for (int k = lane; k < NMAX * SP; k += 32) xs[k] = 0.f;
  __syncthreads();

  const bool vec_x = ((S & 3) == 0) && a.x_vec;
  const bool vec_y = ((S & 3) == 0) && ((H & 3) == 0);
  const int64_t b_begin = (int64_t)blockIdx.x * wins_per_cta;
  int64_t b_end = b_begin + wins_per_cta;
  if (b_end > a.B) b_end = a.B;

  for (int64_t b = b_begin + warp; b < b_end; b += nwarps) {
    const int64_t series = b * C + c;
    // ---------------- a1: load + segment (each element read once)
    const float* xg = a.x + b * a.xsb + c * a.xsc + a.r;
    if (vec_x) {
      const int n4 = (N * S) >> 2;  // SP == S: rows are contiguous
      for (int k = lane; k < n4; k += 32)
        reinterpret_cast<float4*>(xs)[k] = ldg_stream4(xg + 4 * k);
    } else {
      for (int k = lane; k < N * S; k += 32) {
        int n = k / S, t = k - n * S;
        xs[n * SP + t] = __ldg(xg + k);
      }
    }
    __syncwarp();

    // ---------------- a2: descriptors of segment i = lane (shifted by its first value,
    // so a constant segment gives z = 0 exactly, as the fp64 definition does)
    const int i = lane;
    float mu = 0.f, nu2 = 0.f, kap = 0.f, inv = 0.f;
    if (i < N) {
      const float* xr = xs + i * SP;
      const float x0 = xr[0];
      float s = 0.f;
      for (int t = 0; t < S; t++) s += xr[t] - x0;
      const float m1 = s * a.inv_s;
      mu = x0 + m1;
      for (int t = 0; t < S; t++) {
        const float z = (xr[t] - x0) - m1;
        nu2 = fmaf(z, z, nu2);
        kap = fmaf((float)t - a.half_s, z, kap);
        zt[t * NMAX + i] = z;
      }
      kap *= a.inv_v;
      inv = rsqrtf(nu2 + kEpsSeasonal);
    } else if (i < NMAX) {
      for (int t = 0; t < S; t++) zt[t * NMAX + i] = 0.f;
    }
    const float mbar = warp_sum(i < N ? mu : 0.f) * a.inv_n;
    const float dv = i < N ? nu2 + (float)S * (mu - mbar) * (mu - mbar) : 0.f;
    const float sigma2 = warp_sum(dv) * a.inv_ns;
    const float inv_var = 1.0f / (sigma2 + kEpsTrend);
    __syncwarp();

    // ---------------- a3: seasonal Gram row i (z_j broadcast as float4)
    float acc[NMAX];
#pragma unroll
    for (int j = 0; j < NMAX; j++) acc[j] = 0.f;
    if (i < NMAX) {
      for (int t = 0; t < S; t++) {
        const float zi = zt[t * NMAX + i];
        const float4* zr = reinterpret_cast<const float4*>(zt + t * NMAX);
#pragma unroll
        for (int j4 = 0; j4 < NMAX / 4; j4++) {
          const float4 v = zr[j4];
          acc[4 * j4 + 0] = fmaf(zi, v.x, acc[4 * j4 + 0]);
          acc[4 * j4 + 1] = fmaf(zi, v.y, acc[4 * j4 + 1]);
          acc[4 * j4 + 2] = fmaf(zi, v.z, acc[4 * j4 + 2]);
          acc[4 * j4 + 3] = fmaf(zi, v.w, acc[4 * j4 + 3]);
        }
      }
    }

    // ---------------- a5 (seasonal): rho_ij = G_ij inv_i inv_j; row softmax
    {
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < NMAX; j++) {
        const float invj = __shfl_sync(0xffffffffu, inv, j);
        acc[j] = j < N ? acc[j] * inv * invj : -INFINITY;
        mx = fmaxf(mx, acc[j]);
      }
      float sum = 0.f;
#pragma unroll
      for (int j = 0; j < NMAX; j++) {
        acc[j] = j < N ? fast_ex2((acc[j] - mx) * a.ks) : 0.f;
        sum += acc[j];
      }
      const float rs = 1.0f / sum;
      if (i < NMAX) {
#pragma unroll
        for (int j = 0; j < NMAX; j++) as_[i * AP + j] = i < N ? acc[j] * rs : 0.f;
      }
      if (a.a_s_dbg != nullptr && i < N) {
        float* d = a.a_s_dbg + (series * N + i) * N;
#pragma unroll
        for (int j = 0; j < NMAX; j++)
          if (j < N) d[j] = acc[j] * rs;
      }
    }
    // ---------------- a4 + a5 (trend): Dhat_ij, row softmax of -Dhat / tau_t
    {
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < NMAX; j++) {
        const float muj = __shfl_sync(0xffffffffu, mu, j);
        const float kj = __shfl_sync(0xffffffffu, kap, j);
        const float dm = mu - muj, dk = kap - kj;
        const float d = fmaf(a.vtrend * dk, dk, dm * dm) * inv_var;
        acc[j] = j < N ? -d : -INFINITY;
        mx = fmaxf(mx, acc[j]);
      }
      float sum = 0.f;
#pragma unroll
      for (int j = 0; j < NMAX; j++) {
        acc[j] = j < N ? fast_ex2((acc[j] - mx) * a.kt) : 0.f;
        sum += acc[j];
      }
      const float rs = 1.0f / sum;
      if (i < NMAX) {
#pragma unroll
        for (int j = 0; j < NMAX; j++) at_[i * AP + j] = i < N ? acc[j] * rs : 0.f;
      }
      if (a.a_t_dbg != nullptr && i < N) {
        float* d = a.a_t_dbg + (series * N + i) * N;
#pragma unroll
        for (int j = 0; j < NMAX; j++)
          if (j < N) d[j] = acc[j] * rs;
      }
    }
    __syncwarp();

    // ---------------- a6+a7 (fold): lane j holds columns A_s[:, j], A_t[:, j];
    // Q[m][j] = sum_i W_s[m][i] A_s[i][j] + W_t[m][i] A_t[i][j]
    if (lane < NMAX) {
      const int j = lane;
      float cs[NMAX], ct[NMAX];
#pragma unroll
      for (int ii = 0; ii < NMAX; ii++) {
        cs[ii] = as_[ii * AP + j];
        ct[ii] = at_[ii * AP + j];
      }
      for (int m = 0; m < M; m++) {
        const float4* w4s = reinterpret_cast<const float4*>(wsS + m * NMAX);
        const float4* w4t = reinterpret_cast<const float4*>(wtS + m * NMAX);
        float q = 0.f;
#pragma unroll
        for (int k4 = 0; k4 < NMAX / 4; k4++) {
          const float4 u = w4s[k4], v = w4t[k4];
          q = fmaf(u.x, cs[4 * k4 + 0], q);
          q = fmaf(u.y, cs[4 * k4 + 1], q);
          q = fmaf(u.z, cs[4 * k4 + 2], q);
          q = fmaf(u.w, cs[4 * k4 + 3], q);
          q = fmaf(v.x, ct[4 * k4 + 0], q);
          q = fmaf(v.y, ct[4 * k4 + 1], q);
          q = fmaf(v.z, ct[4 * k4 + 2], q);
          q = fmaf(v.w, ct[4 * k4 + 3], q);
        }
        qs[m * QP + j] = q;
      }
    }
    __syncwarp();

    // ---------------- a7: Y[m][t] = sum_j Q[m][j] X[j][t]  (lane m; X rows broadcast)
    for (int m = lane; m < M; m += 32) {
      float q[NMAX];
#pragma unroll
      for (int j = 0; j < NMAX; j++) q[j] = qs[m * QP + j];
      for (int t4 = 0; t4 < SP; t4 += 4) {
        float4 yv = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < NMAX; j++) {
          const float4 xv = *reinterpret_cast<const float4*>(xs + j * SP + t4);
          yv.x = fmaf(q[j], xv.x, yv.x);
          yv.y = fmaf(q[j], xv.y, yv.y);
          yv.z = fmaf(q[j], xv.z, yv.z);
          yv.w = fmaf(q[j], xv.w, yv.w);
        }
        float* yr = ys + m * YP + t4;
        yr[0] = yv.x;
        if (t4 + 1 < S) yr[1] = yv.y;
        if (t4 + 2 < S) yr[2] = yv.z;
        if (t4 + 3 < S) yr[3] = yv.w;
      }
    }
    __syncwarp();

    // ---------------- a8: y[h] = Y[h / S][h % S] + b[h]  (coalesced)
    float* yg = a.y + series * H;
    if (vec_y) {
      for (int h = 4 * lane; h < H; h += 128) {
        const int m = h / S, t = h - m * S;  // S % 4 == 0: the 4 steps share m
        const float* yr = ys + m * YP + t;
        float4 v;
        v.x = yr[0] + bS[h];
        v.y = yr[1] + bS[h + 1];
        v.z = yr[2] + bS[h + 2];
        v.w = yr[3] + bS[h + 3];
        stg_stream4(yg + h, v);
      }
    } else {
      for (int h = lane; h < H; h += 32) {
        const int m = h / S, t = h - m * S;
        yg[h] = ys[m * YP + t] + bS[h];
      }
    }
    __syncwarp();
  }
}

static int round4(int v) { return (v + 3) & ~3; }

bool plan_warp_kernel(const FwdArgs& a, int max_smem_optin, WarpPlan* p) {
  if (a.N > 32) return false;
  p->nmax = a.N <= 8 ? 8 : (a.N <= 16 ? 16 : 32);
  const int nmax = p->nmax;
  const int SP = (a.S + 3) & ~3;
  const int YP = a.S | 1;
  const int r1 = nmax * SP;
  const int r2 = a.S * nmax > a.M * (nmax + 1) ? a.S * nmax : a.M * (nmax + 1);
  const int r3a = 2 * nmax * (nmax + 1), r3b = a.M * YP;
  const int r3 = r3a > r3b ? r3a : r3b;
  p->off_r2 = round4(r1);
  p->off_r3 = p->off_r2 + round4(r2);
  p->per_warp_floats = p->off_r3 + round4(r3);
  p->shared_floats = round4(2 * a.M * nmax + a.H);
  // 4 warps per CTA keeps ~2-3 CTAs resident per SM at the Traffic shape.
  p->warps_per_cta = 4;
  p->smem_bytes =
      (size_t)(p->shared_floats + p->warps_per_cta * p->per_warp_floats) * sizeof(float);
  while (p->smem_bytes > (size_t)max_smem_optin && p->warps_per_cta > 1) {
    p->warps_per_cta >>= 1;
    p->smem_bytes =
        (size_t)(p->shared_floats + p->warps_per_cta * p->per_warp_floats) * sizeof(float);
  }
  if (p->smem_bytes > (size_t)max_smem_optin) return false;
  // windows per CTA: amortise the per-channel head staging over 4 series per warp
  p->wins_per_cta = p->warps_per_cta * 4;
  return true;
}

template <int NMAX>
static cudaError_t launch_t(const FwdArgs& a, const WarpPlan& p, cudaStream_t st) {
  auto k = prnet_fwd_warp_kernel<NMAX>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((a.B + p.wins_per_cta - 1) / p.wins_per_cta), (unsigned)a.C);
  dim3 block(32 * p.warps_per_cta);
  k<<<grid, block, p.smem_bytes, st>>>(a, p.wins_per_cta, p.per_warp_floats, p.off_r2, p.off_r3,
                                       p.shared_floats);
  return cudaGetLastError();
}

cudaError_t launch_warp_kernel(const FwdArgs& a, const WarpPlan& p, cudaStream_t st) {
  switch (p.nmax) {
    case 8: return launch_t<8>(a, p, st);
    case 16: return launch_t<16>(a, p, st);
    default: return launch_t<32>(a, p, st);
  }
}

}  // namespace prnet
