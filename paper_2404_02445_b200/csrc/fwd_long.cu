// fwd_long.cu -- fused PRNet pattern-attention forward for 32 < N <= 512
// segments per series (the long-lookback points of the stress sweep,
// BASELINE.json configs[4]: L up to 5760, S down to 12 -> N up to 480).
//
// The N x N similarity matrices no longer fit a warp's registers, and at
// N = 480 not even shared memory (2 x 922 KB), so the kernel streams rows:
// one CTA owns one series; warp w takes query rows i = w, w + nwarps, ...;
// for row i the lanes cover the keys j = lane + 32 k, compute the row's
// seasonal and trend logits, softmax them with warp reductions, aggregate
// the pattern rows P_s[i][:], P_t[i][:] (Def 9) and immediately fold them
// into the head accumulator Y[m][t] += W_s[m][i] P_s[i][t] + W_t[m][i] P_t[i][t]
// (Def 10) kept per warp in shared memory.  A fixed-order reduction over the
// warps then adds the bias (Def 11).  The same reading and the
// same step map as fwd_warp.cu.
#include "prnet_internal.cuh"

namespace prnet {

template <int KJ>
__global__ void __launch_bounds__(256) prnet_fwd_long_kernel(FwdArgs a, int rs) {
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int S = a.S, N = a.N, M = a.M, H = a.H, C = a.C;
  const int MS = M * S;

  float* xr = smem;               // [N][rs]  segments, odd row stride
  float* zr = xr + N * rs;        // [N][rs]  z
  float* muS = zr + N * rs;       // [N]
  float* kapS = muS + N;          // [N]
  float* invS = kapS + N;         // [N]
  float* red = invS + N;          // [64]     block reduction scratch
  float* wrow = red + 64;         // [nwarps][2][N]  softmax rows
  float* yw = wrow + nwarps * 2 * N;  // [nwarps][M*S] per-warp head accumulators
  float* muZ = yw + nwarps * MS;      // [N] seasonal-branch level (= muS unless ma_kernel)
  float* kapZ = muZ + N;              // [N] seasonal-branch slope
  float* trr = kapZ + N;              // [N][rs] trend rows (ma_kernel only)
  const bool dec = a.ma_k > 0;

  const int64_t total = a.B * (int64_t)C;
  for (int64_t series = blockIdx.x; series < total; series += gridDim.x) {
    const int c = (int)(series % C);
    const int cw = a.head_per_channel ? c : 0;
    const float* gws = a.ws + (int64_t)cw * M * N;
    const float* gwt = a.wt + (int64_t)cw * M * N;

    // ---- a1: load + segment
    const float* xg = a.x + (series / C) * a.xsb + c * a.xsc + a.r;
    for (int k = threadIdx.x; k < N * S; k += blockDim.x) {
      const int n = k / S, t = k - n * S;
      xr[n * rs + t] = __ldg(xg + k);
    }
    for (int k = lane; k < MS; k += 32) yw[warp * MS + k] = 0.f;
    __syncthreads();
    // ma_kernel (R-f5): trend = moving average of the N S segmented points (ends repeated),
    // thread-chunked running sums; RevIN statistics of the raw points; then xr holds the
    // seasonal rows x - trend and trr the trend rows
    float dec_mr = 0.f, dec_var = 0.f;
    if (dec) {
      const int NS = N * S, hk = (a.ma_k - 1) >> 1;
      auto xat = [&](int q) {
        q = q < 0 ? 0 : (q > NS - 1 ? NS - 1 : q);
        const int n = q / S;
        return xr[n * rs + (q - n * S)];
      };
      const int cnk = (NS + blockDim.x - 1) / blockDim.x;
      const int i0 = threadIdx.x * cnk, i1 = min(i0 + cnk, NS);
      if (i0 < i1) {
        float sacc = 0.f;
        for (int d = -hk; d <= hk; d++) sacc += xat(i0 + d);
        for (int q = i0; q < i1; q++) {
          if (q > i0) sacc += xat(q + hk) - xat(q - 1 - hk);
          const int n = q / S;
          trr[n * rs + (q - n * S)] = sacc * a.ma_inv;
        }
      }
      float ps = 0.f;
      for (int q = threadIdx.x; q < NS; q += blockDim.x) ps += xat(q);
      ps = warp_sum(ps);
      if (lane == 0) red[warp] = ps;
      __syncthreads();
      for (int w = 0; w < nwarps; w++) dec_mr += red[w];
      dec_mr *= a.inv_ns;
      __syncthreads();
      ps = 0.f;
      for (int q = threadIdx.x; q < NS; q += blockDim.x) {
        const float d = xat(q) - dec_mr;
        ps = fmaf(d, d, ps);
      }
      ps = warp_sum(ps);
      if (lane == 0) red[warp] = ps;
      __syncthreads();
      for (int w = 0; w < nwarps; w++) dec_var += red[w];
      dec_var *= a.inv_ns;
      __syncthreads();
      for (int q = threadIdx.x; q < NS; q += blockDim.x) {
        const int n = q / S, o = n * rs + (q - n * S);
        xr[o] -= trr[o];
      }
      __syncthreads();
    }

    // ---- a2: descriptors, one thread per segment (shifted by the first value); with
    // metric_variant bit 1 the seasonal rows are the residuals e = z - kappa t~ (R-f3)
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
      const float* row = xr + n * rs;
      const float x0 = row[0];
      float s = 0.f, s3 = 0.f;
      for (int t = 0; t < S; t++) {
        const float d = row[t] - x0;
        s += d;
        s3 = fmaf((float)t - a.half_s, d, s3);
      }
      const float m1 = s * a.inv_s;
      const float kap = s3 * a.inv_v;
      const float kd = a.detrend ? kap : 0.f;
      float nu2 = 0.f;
      for (int t = 0; t < S; t++) {
        const float z = fmaf(-kd, (float)t - a.half_s, (row[t] - x0) - m1);
        nu2 = fmaf(z, z, nu2);
        zr[n * rs + t] = z;
      }
      muZ[n] = x0 + m1;
      kapZ[n] = kap;
      invS[n] = nu2;   // seasonal |z|^2 (|e|^2); the normaliser follows the RevIN scale below
      if (!dec) {
        muS[n] = x0 + m1;
        kapS[n] = kap;
        // |z|^2 for sigma^2 (= |e|^2 + kappa^2 V when detrended) in the wrow scratch (free
        // until phase 2)
        wrow[n] = a.detrend ? fmaf(kap * kap, 1.f / a.inv_v, nu2) : nu2;
      } else {   // trend branch: the trend row's level, slope and |z|^2 (sigma^2)
        const float* tr = trr + n * rs;
        const float y0 = tr[0];
        float st = 0.f, st3 = 0.f;
        for (int t = 0; t < S; t++) {
          const float d = tr[t] - y0;
          st += d;
          st3 = fmaf((float)t - a.half_s, d, st3);
        }
        const float mt1 = st * a.inv_s;
        float q2 = 0.f;
        for (int t = 0; t < S; t++) {
          const float z = (tr[t] - y0) - mt1;
          q2 = fmaf(z, z, q2);
        }
        muS[n] = y0 + mt1;
        kapS[n] = st3 * a.inv_v;
        wrow[n] = q2;
      }
    }
    __syncthreads();
    // sigma^2: fixed-order block reduction (deterministic)
    float part = 0.f;
    for (int n = threadIdx.x; n < N; n += blockDim.x) part += muS[n];
    part = warp_sum(part);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    float mbar = 0.f;
    for (int w = 0; w < nwarps; w++) mbar += red[w];
    mbar *= a.inv_n;
    __syncthreads();
    part = 0.f;
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
      const float d = muS[n] - mbar;
      part += wrow[n] + (float)S * d * d;
    }
    part = warp_sum(part);
    if (lane == 0) red[32 + warp] = part;
    __syncthreads();
    float sig = 0.f;
    for (int w = 0; w < nwarps; w++) sig += red[32 + w];
    // instance normalisation (R-f1): every descriptor of xhat = (x - mr) rr is an affine image
    // of the one of x; the patterns are mapped back in a6 (P - mr) and a8 adds sr b + mr
    float mr = 0.f, rr = 1.f, sr = 1.f;
    if (a.revin) {
      const float vr = dec ? dec_var : sig * a.inv_ns;   // of the raw segmented points
      mr = dec ? dec_mr : mbar;
      rr = rsqrtf(vr + kEpsRevin);
      sr = (vr + kEpsRevin) * rr;
    }
    // trend: D^ of xhat = rr^2 D / (var rr^2 + eps_t)
    const float inv_var = rr * rr / fmaf(sig * a.inv_ns * rr, rr, kEpsTrend);
    __syncthreads();  // wrow scratch is reused below
    for (int n = threadIdx.x; n < N; n += blockDim.x)
      invS[n] = rsqrtf(invS[n] * rr * rr + kEpsSeasonal) * rr;   // rho of xhat
    __syncthreads();

    // ---- a3..a7 streamed over query rows
    float* wr = wrow + warp * 2 * N;
    for (int i = warp; i < N; i += nwarps) {
      float g[KJ];
#pragma unroll
      for (int k = 0; k < KJ; k++) g[k] = 0.f;
      const float* zi = zr + i * rs;
      for (int t = 0; t < S; t++) {
        const float zv = zi[t];
#pragma unroll
        for (int k = 0; k < KJ; k++) {
          const int j = lane + 32 * k;
          if (j < N) g[k] = fmaf(zv, zr[j * rs + t], g[k]);
        }
      }
      const float inv_i = invS[i], mu_i = muS[i], k_i = kapS[i];
      // seasonal softmax
      float mx = -INFINITY;
#pragma unroll
      for (int k = 0; k < KJ; k++) {
        const int j = lane + 32 * k;
        g[k] = j < N ? g[k] * inv_i * invS[j] : -INFINITY;
        mx = fmaxf(mx, g[k]);
      }
      mx = warp_max(mx);
      float sum = 0.f;
#pragma unroll
      for (int k = 0; k < KJ; k++) {
        const int j = lane + 32 * k;
        g[k] = j < N ? fast_ex2((g[k] - mx) * a.ks) : 0.f;
        sum += g[k];
      }
      float rsum = 1.0f / warp_sum(sum);
#pragma unroll
      for (int k = 0; k < KJ; k++) {
        const int j = lane + 32 * k;
        if (j < N) wr[j] = g[k] * rsum;
        if (a.a_s_dbg != nullptr && j < N) a.a_s_dbg[(series * N + i) * N + j] = g[k] * rsum;
      }
      // trend softmax
      mx = -INFINITY;
#pragma unroll
      for (int k = 0; k < KJ; k++) {
        const int j = lane + 32 * k;
        float v = -INFINITY;
        if (j < N) {
          const float dm = mu_i - muS[j], dk = k_i - kapS[j];
          v = -(fmaf(a.vtrend * dk, dk, dm * dm) * inv_var);   // kapS: slope (x units)
        }
        g[k] = v;
        mx = fmaxf(mx, v);
      }
      mx = warp_max(mx);
      sum = 0.f;
#pragma unroll
      for (int k = 0; k < KJ; k++) {
        const int j = lane + 32 * k;
        g[k] = j < N ? fast_ex2((g[k] - mx) * a.kt) : 0.f;
        sum += g[k];
      }
      rsum = 1.0f / warp_sum(sum);
#pragma unroll
      for (int k = 0; k < KJ; k++) {
        const int j = lane + 32 * k;
        if (j < N) wr[N + j] = g[k] * rsum;
        if (a.a_t_dbg != nullptr && j < N) a.a_t_dbg[(series * N + i) * N + j] = g[k] * rsum;
      }
      __syncwarp();
      // component values (metric_variant bit 2, R-f4): row sums A mu, A kappa of both branches
      float asm_ = 0.f, ask = 0.f, atm = 0.f, atk = 0.f;
      if (a.comp) {
        for (int j = lane; j < N; j += 32) {
          asm_ = fmaf(wr[j], muZ[j], asm_);
          ask = fmaf(wr[j], kapZ[j], ask);
          atm = fmaf(wr[N + j], muS[j], atm);
          atk = fmaf(wr[N + j], kapS[j], atk);
        }
        asm_ = warp_sum(asm_);
        ask = warp_sum(ask) * (a.detrend ? 1.f : 0.f);
        atm = warp_sum(atm);
        atk = warp_sum(atk) * (a.vtrend != 0.f ? 1.f : 0.f);
      }
      // a6: P_s[i][t], P_t[i][t] by lane t; a7: fold row i into Y
      for (int t = lane; t < S; t += 32) {
        float ps = 0.f, pt = 0.f;
        const float* tx = dec ? trr : xr;   // trend-branch rows
        for (int j = 0; j < N; j++) {
          ps = fmaf(wr[j], xr[j * rs + t], ps);
          pt = fmaf(wr[N + j], tx[j * rs + t], pt);
        }
        if (a.comp) {
          // P_s = A (x - mu - d1 kappa t~), P_t = A (mu + d0 kappa t~)
          const float tt = (float)t - a.half_s;
          ps = ps - fmaf(ask, tt, asm_);
          pt = fmaf(atk, tt, atm);
        }
        // RevIN: rows of A sum to 1, so A xhat = rr (A x - mr) (rr sr = 1); only the branches
        // that carry the level (both for the raw reading, the trend one for component values
        // or the decomposition) shift by mr
        if (!(a.comp || dec)) ps -= mr;
        pt -= mr;
        float* yr = yw + warp * MS + t;
        for (int m = 0; m < M; m++)
          yr[m * S] = fmaf(__ldg(gws + m * N + i), ps, fmaf(__ldg(gwt + m * N + i), pt, yr[m * S]));
      }
      __syncwarp();
    }
    __syncthreads();
    // ---- a8: fixed-order reduction over warps + bias
    const float* gb = a.bias + (int64_t)cw * H;
    float* yg = a.y + series * H;
    for (int h = threadIdx.x; h < H; h += blockDim.x) {
      float v = 0.f;
      for (int w = 0; w < nwarps; w++) v += yw[w * MS + h];
      yg[h] = v + fmaf(gb[h], sr, mr);
    }
    __syncthreads();
  }
}

bool plan_long_kernel(const FwdArgs& a, int max_smem_optin, int sm_count, LongPlan* p) {
  if (a.N > 512) return false;
  p->kjmax = a.N <= 64 ? 2 : (a.N <= 128 ? 4 : (a.N <= 256 ? 8 : 16));
  p->rs = a.S | 1;
  p->warps_per_cta = 8;
  const size_t floats = (size_t)2 * a.N * p->rs + 3 * a.N + 64 +
                        (size_t)p->warps_per_cta * (2 * a.N + a.M * a.S) + 2 * a.N +
                        (a.ma_k > 0 ? (size_t)a.N * p->rs : 0);
  p->smem_bytes = floats * sizeof(float);
  if (p->smem_bytes > (size_t)max_smem_optin) return false;
  const int64_t total = a.B * (int64_t)a.C;
  int per_sm = (int)((228 * 1024) / (p->smem_bytes + 1024));
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 8) per_sm = 8;
  int64_t g = (int64_t)sm_count * per_sm;
  p->grid = (int)(total < g ? total : g);
  if (p->grid < 1) p->grid = 1;
  return true;
}

template <int KJ>
static cudaError_t launch_t(const FwdArgs& a, const LongPlan& p, cudaStream_t st) {
  auto k = prnet_fwd_long_kernel<KJ>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  k<<<p.grid, 32 * p.warps_per_cta, p.smem_bytes, st>>>(a, p.rs);
  return cudaGetLastError();
}

cudaError_t launch_long_kernel(const FwdArgs& a, const LongPlan& p, cudaStream_t st) {
  switch (p.kjmax) {
    case 2: return launch_t<2>(a, p, st);
    case 4: return launch_t<4>(a, p, st);
    case 8: return launch_t<8>(a, p, st);
    default: return launch_t<16>(a, p, st);
  }
}

}  // namespace prnet
