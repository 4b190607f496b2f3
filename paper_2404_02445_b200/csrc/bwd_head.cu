// bwd_head.cu -- backward pass of the PRNet head (reading R-f6 in
// DESIGN.md §3): for an upstream gradient dy = dL/dy,
//   dY[m][t] = dy[m S + t] s_r (0 past H),  dW_s[m][n] = sum_{series, t} dY[m][t] P_s[n][t],
//   dW_t likewise with P_t,  db[h] = sum_series dy[h] s_r,
// summed over the batch (and over the channels for a shared head).  The head enters y
// linearly, so the gradients need the patterns P = A X̂ of every series but not W: the
// kernel recomputes descriptors, both attentions and the patterns in FP32 (same reading as
// the forward kernels, with every flag but component values and the decomposition).
//
// Layout: one warp per series, lane i = segment i (N <= 32), 8 warps (fewer for long
// segments) per CTA, one channel per CTA.  Per-warp shared memory: X, Z [S][NP] and dY
// [S][MP] (transposed, zero-padded), the bias gradient [H].  Lane i keeps its
// column of dW_s, dW_t ([M] each) in registers over all the warp's series; at the end the
// warps are reduced in a fixed order into one partial per CTA, and prnet_bwd_reduce sums the
// partials in fp64 in a fixed order.  Deterministic, no atomics.
#include <algorithm>
#include <cstdlib>

#include "prnet_internal.cuh"

namespace prnet {

namespace {

__device__ __forceinline__ float shfl(float v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

// NP / MP: segment / future-segment counts padded to 8, 16 or 32.  X, Z and dY are stored
// transposed ([t][NP], [t][MP]) with zero padding rows, so every inner loop is unguarded,
// a row of all segments at one t is NP/4 broadcast float4 loads, and lane i's own element
// at t is conflict-free.
template <int NP, int MP>
__global__ void __launch_bounds__(384, 1) prnet_bwd_head_kernel(FwdArgs a, const float* __restrict__ dy,
                                                          float* __restrict__ part,
                                                          BwdLayout ly) {
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int c = blockIdx.y, C = a.C;
  const int N = a.N, S = a.S, M = a.M, H = a.H;
  float* wbase = smem + warp * ly.per_warp;
  float* X = wbase;                      // [S][NP]
  float* Z = X + S * NP;                 // [S][NP]
  float* dYs = wbase + ly.off_dy;        // [S][MP]
  float* accB = wbase + ly.off_db;       // [H]
  for (int k = lane; k < H; k += 32) accB[k] = 0.f;
  for (int k = lane; k < 2 * S * NP; k += 32) X[k] = 0.f;   // padding rows stay 0
  for (int k = lane; k < S * MP; k += 32) dYs[k] = 0.f;

  const int i = lane;
  float accS[MP], accT[MP];   // lane i: dW_s[m][i], dW_t[m][i]
#pragma unroll
  for (int m = 0; m < MP; m++) accS[m] = accT[m] = 0.f;

  const int64_t b0 = (int64_t)blockIdx.x * ly.wins_per_cta;
  int64_t b1 = b0 + ly.wins_per_cta;
  if (b1 > a.B) b1 = a.B;
  for (int64_t b = b0 + warp; b < b1; b += nwarps) {
    const int64_t series = b * C + c;
    const float* xg = a.x + b * a.xsb + c * a.xsc + a.r;
    const float* g = dy + series * H;
    __syncwarp();
    // lane = segment row (global reads are L1-served), transposed conflict-free stores
    for (int t = 0; t < S; t++) {
      if (i < N) X[t * NP + i] = __ldg(xg + i * S + t);
      if (i < M) {
        const int h = i * S + t;
        dYs[t * MP + i] = h < H ? __ldg(g + h) : 0.f;
      }
    }
    __syncwarp();

    // a2: descriptors from d = x - x0 (Def 3-4), residual norm with metric_variant bit 1
    float x0 = 0.f, m1 = 0.f, mu = 0.f, kap = 0.f, nu2 = 0.f;
    if (i < N) {
      x0 = X[i];
      float s1 = 0.f, s3 = 0.f;
      for (int t = 0; t < S; t++) {
        const float d = X[t * NP + i] - x0;
        s1 += d;
        s3 = fmaf((float)t - a.half_s, d, s3);
      }
      m1 = s1 * a.inv_s;
      mu = x0 + m1;
      kap = s3 * a.inv_v;
      const float kd = a.detrend ? kap : 0.f;
      for (int t = 0; t < S; t++) {
        const float z = fmaf(-kd, (float)t - a.half_s, (X[t * NP + i] - x0) - m1);
        Z[t * NP + i] = z;
        nu2 = fmaf(z, z, nu2);
      }
    }
    // Def 5 (|z|^2 = |e|^2 + kappa^2 V when detrended) and the RevIN map (R-f1)
    const float mbar = warp_sum(i < N ? mu : 0.f) * a.inv_n;
    const float nz2 = a.detrend ? fmaf(kap * kap, 1.f / a.inv_v, nu2) : nu2;
    const float var =
        warp_sum(i < N ? nz2 + (float)S * (mu - mbar) * (mu - mbar) : 0.f) * a.inv_ns;
    float mr = 0.f, rr = 1.f, sr = 1.f;
    if (a.revin) {
      mr = mbar;
      rr = rsqrtf(var + kEpsRevin);
      sr = (var + kEpsRevin) * rr;
    }
    const float inv_var = 1.f / fmaf(var * rr, rr, kEpsTrend);
    const float cm = sqrtf(inv_var * a.kt) * rr, ck = sqrtf(a.vtrend * inv_var * a.kt) * rr;
    const float mt = (mu - mr) * cm, kt = kap * ck;                 // trend coordinates
    const float inv = rsqrtf(nu2 * rr * rr + kEpsSeasonal) * rr;    // seasonal normaliser
    __syncwarp();   // Z written

    // a3: Gram row i (padding rows of Z are 0)
    float as[NP], at[NP];
#pragma unroll
    for (int j = 0; j < NP; j++) as[j] = 0.f;
    for (int t = 0; t < S; t++) {
      const float v = Z[t * NP + i];
      const float4* zr = reinterpret_cast<const float4*>(Z + t * NP);
#pragma unroll
      for (int q = 0; q < NP / 4; q++) {
        const float4 z4 = zr[q];
        as[4 * q] = fmaf(v, z4.x, as[4 * q]);
        as[4 * q + 1] = fmaf(v, z4.y, as[4 * q + 1]);
        as[4 * q + 2] = fmaf(v, z4.z, as[4 * q + 2]);
        as[4 * q + 3] = fmaf(v, z4.w, as[4 * q + 3]);
      }
    }
    // a4 + a5: exponents (masked past N), searched row maxima, both softmaxes
    float smax = -INFINITY, tmax = -INFINITY;
#pragma unroll
    for (int j = 0; j < NP; j++) {
      const float invj = shfl(inv, j), mtj = shfl(mt, j), ktj = shfl(kt, j);
      const float dm = mt - mtj, dk = kt - ktj;
      as[j] = j < N ? as[j] * inv * invj * a.ks : -INFINITY;
      at[j] = j < N ? -fmaf(dm, dm, dk * dk) : -INFINITY;
      smax = fmaxf(smax, as[j]);
      tmax = fmaxf(tmax, at[j]);
    }
    float ssum = 0.f, tsum = 0.f;
#pragma unroll
    for (int j = 0; j < NP; j++) {
      as[j] = exp2f(as[j] - smax);
      at[j] = exp2f(at[j] - tmax);
      ssum += as[j];
      tsum += at[j];
    }
    // rows of A sum to 1: P^ = rr (A X - mr); the s_r of dY folded into the row scale
    const float rs = rr * sr / ssum, rt = rr * sr / tsum, off = mr * rr * sr;

    // a6 + gradient: dW[m][i] += sum_t dY[m][t] s_r P^[i][t]
    for (int t = 0; t < S; t++) {
      float ps = 0.f, pt = 0.f;
      const float4* xr = reinterpret_cast<const float4*>(X + t * NP);
#pragma unroll
      for (int q = 0; q < NP / 4; q++) {
        const float4 x4 = xr[q];
        ps = fmaf(as[4 * q], x4.x, ps);
        pt = fmaf(at[4 * q], x4.x, pt);
        ps = fmaf(as[4 * q + 1], x4.y, ps);
        pt = fmaf(at[4 * q + 1], x4.y, pt);
        ps = fmaf(as[4 * q + 2], x4.z, ps);
        pt = fmaf(at[4 * q + 2], x4.z, pt);
        ps = fmaf(as[4 * q + 3], x4.w, ps);
        pt = fmaf(at[4 * q + 3], x4.w, pt);
      }
      ps = fmaf(ps, rs, -off);
      pt = fmaf(pt, rt, -off);
      const float4* gr = reinterpret_cast<const float4*>(dYs + t * MP);
#pragma unroll
      for (int q = 0; q < MP / 4; q++) {
        const float4 g4 = gr[q];
        accS[4 * q] = fmaf(g4.x, ps, accS[4 * q]);
        accT[4 * q] = fmaf(g4.x, pt, accT[4 * q]);
        accS[4 * q + 1] = fmaf(g4.y, ps, accS[4 * q + 1]);
        accT[4 * q + 1] = fmaf(g4.y, pt, accT[4 * q + 1]);
        accS[4 * q + 2] = fmaf(g4.z, ps, accS[4 * q + 2]);
        accT[4 * q + 2] = fmaf(g4.z, pt, accT[4 * q + 2]);
        accS[4 * q + 3] = fmaf(g4.w, ps, accS[4 * q + 3]);
        accT[4 * q + 3] = fmaf(g4.w, pt, accT[4 * q + 3]);
      }
    }
    for (int k = lane; k < H; k += 32) {
      const int m = k / S;
      accB[k] = fmaf(dYs[(k - m * S) * MP + m], sr, accB[k]);
    }
  }

  // fixed-order reduction over the warps into this CTA's partial [dW_s | dW_t | db]
  // (lanes past N hold padding columns and are not read)
  __syncthreads();
  float* red = smem + warp * ly.per_warp;   // reuse the X region: [2][M][32]
#pragma unroll
  for (int m = 0; m < MP; m++) {
    if (m < M) {
      red[m * 32 + lane] = accS[m];
      red[(M + m) * 32 + lane] = accT[m];
    }
  }
  __syncthreads();
  const int MN = M * N, E = 2 * MN + H;
  float* out = part + ((int64_t)c * gridDim.x + blockIdx.x) * E;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    float v = 0.f;
    if (e < 2 * MN) {
      const int br = e / MN, mn = e - br * MN, m = mn / N, n = mn - m * N;
      for (int w = 0; w < nwarps; w++) v += smem[w * ly.per_warp + (br * M + m) * 32 + n];
    } else {
      const int hh = e - 2 * MN;
      for (int w = 0; w < nwarps; w++) v += smem[w * ly.per_warp + ly.off_db + hh];
    }
    out[e] = v;
  }
}

// out[cw][e] = sum over the channels of cw (all of them for a shared head) and the CTA
// partials, in fp64, in a fixed order
__global__ void prnet_bwd_reduce_kernel(const float* __restrict__ part, int C, int nblk, int E,
                                        int MN, int H, int hpc, float* dws, float* dwt,
                                        float* db) {
  const int cw = blockIdx.y;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    double v = 0.0;
    const int c0 = hpc ? cw : 0, c1 = hpc ? cw + 1 : C;
    for (int c = c0; c < c1; c++)
      for (int k = 0; k < nblk; k++) v += (double)part[((int64_t)c * nblk + k) * E + e];
    if (e < MN) dws[(int64_t)cw * MN + e] = (float)v;
    else if (e < 2 * MN) dwt[(int64_t)cw * MN + e - MN] = (float)v;
    else db[(int64_t)cw * H + e - 2 * MN] = (float)v;
  }
}

// Long lookbacks (32 < N <= 512): one CTA per (channel, block of windows), series one after
// the other; per series the segment rows, z rows and dY live in shared memory, warp w takes
// query rows i = w, w + nwarps, ... (as fwd_long.cu): the row's two softmaxes over the keys
// (lanes over j), its pattern row P^[i][t] (lanes over t), and dW[m][i] += sum_t dY[m][t] P^
// by a warp reduction per m into the CTA's accumulator (row i has one owner warp: no atomics).
template <int KJ>
__global__ void __launch_bounds__(256) prnet_bwd_long_kernel(FwdArgs a, const float* __restrict__ dy,
                                                          float* __restrict__ part, int rs,
                                                          int wins_per_cta) {
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int c = blockIdx.y, C = a.C;
  const int S = a.S, N = a.N, M = a.M, H = a.H, MS = M * S;
  float* xr = smem;               // [N][rs]
  float* zr = xr + N * rs;        // [N][rs]
  float* muS = zr + N * rs;       // [N]
  float* kapS = muS + N;          // [N]
  float* invS = kapS + N;         // [N]
  float* red = invS + N;          // [64]
  float* wrow = red + 64;         // [nwarps][2][N]
  float* dYs = wrow + nwarps * 2 * N;   // [M S]
  float* acc = dYs + MS;          // [2][M][N] dW_s, dW_t
  float* accB = acc + 2 * M * N;  // [H]
  for (int k = threadIdx.x; k < 2 * M * N; k += blockDim.x) acc[k] = 0.f;
  for (int k = threadIdx.x; k < H; k += blockDim.x) accB[k] = 0.f;

  const int64_t b0 = (int64_t)blockIdx.x * wins_per_cta;
  int64_t b1 = b0 + wins_per_cta;
  if (b1 > a.B) b1 = a.B;
  for (int64_t b = b0; b < b1; b++) {
    const int64_t series = b * C + c;
    const float* xg = a.x + b * a.xsb + c * a.xsc + a.r;
    __syncthreads();
    for (int k = threadIdx.x; k < N * S; k += blockDim.x) {
      const int n = k / S;
      xr[n * rs + (k - n * S)] = __ldg(xg + k);
    }
    for (int k = threadIdx.x; k < MS; k += blockDim.x) dYs[k] = k < H ? __ldg(dy + series * H + k) : 0.f;
    __syncthreads();
    // descriptors (Def 3-4, residuals with metric_variant bit 1), as fwd_long.cu
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
      const float* row = xr + n * rs;
      const float x0 = row[0];
      float s1 = 0.f, s3 = 0.f;
      for (int t = 0; t < S; t++) {
        const float d = row[t] - x0;
        s1 += d;
        s3 = fmaf((float)t - a.half_s, d, s3);
      }
      const float m1 = s1 * a.inv_s, kap = s3 * a.inv_v, kd = a.detrend ? kap : 0.f;
      float nu2 = 0.f;
      for (int t = 0; t < S; t++) {
        const float z = fmaf(-kd, (float)t - a.half_s, (row[t] - x0) - m1);
        nu2 = fmaf(z, z, nu2);
        zr[n * rs + t] = z;
      }
      muS[n] = x0 + m1;
      kapS[n] = kap;
      invS[n] = nu2;
      wrow[n] = a.detrend ? fmaf(kap * kap, 1.f / a.inv_v, nu2) : nu2;
    }
    __syncthreads();
    float p0 = 0.f;
    for (int n = threadIdx.x; n < N; n += blockDim.x) p0 += muS[n];
    p0 = warp_sum(p0);
    if (lane == 0) red[warp] = p0;
    __syncthreads();
    float mbar = 0.f;
    for (int w = 0; w < nwarps; w++) mbar += red[w];
    mbar *= a.inv_n;
    __syncthreads();
    p0 = 0.f;
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
      const float d = muS[n] - mbar;
      p0 += wrow[n] + (float)S * d * d;
    }
    p0 = warp_sum(p0);
    if (lane == 0) red[32 + warp] = p0;
    __syncthreads();
    float sig = 0.f;
    for (int w = 0; w < nwarps; w++) sig += red[32 + w];
    float mr = 0.f, rr = 1.f, sr = 1.f;
    if (a.revin) {
      const float vr = sig * a.inv_ns;
      mr = mbar;
      rr = rsqrtf(vr + kEpsRevin);
      sr = (vr + kEpsRevin) * rr;
    }
    const float inv_var = rr * rr / fmaf(sig * a.inv_ns * rr, rr, kEpsTrend);
    __syncthreads();
    for (int n = threadIdx.x; n < N; n += blockDim.x)
      invS[n] = rsqrtf(invS[n] * rr * rr + kEpsSeasonal) * rr;
    __syncthreads();

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
      float mx = -INFINITY;
#pragma unroll
      for (int k = 0; k < KJ; k++) {
        const int j = lane + 32 * k;
        g[k] = j < N ? g[k] * inv_i * invS[j] * a.ks : -INFINITY;
        mx = fmaxf(mx, g[k]);
      }
      mx = warp_max(mx);
      float sum = 0.f;
#pragma unroll
      for (int k = 0; k < KJ; k++) {
        const int j = lane + 32 * k;
        g[k] = j < N ? exp2f(g[k] - mx) : 0.f;
        sum += g[k];
      }
      float rsum = 1.f / warp_sum(sum);
#pragma unroll
      for (int k = 0; k < KJ; k++) {
        const int j = lane + 32 * k;
        if (j < N) wr[j] = g[k] * rsum;
      }
      mx = -INFINITY;
#pragma unroll
      for (int k = 0; k < KJ; k++) {
        const int j = lane + 32 * k;
        float v = -INFINITY;
        if (j < N) {
          const float dm = mu_i - muS[j], dk = k_i - kapS[j];
          v = -(fmaf(a.vtrend * dk, dk, dm * dm) * inv_var) * a.kt;
        }
        g[k] = v;
        mx = fmaxf(mx, v);
      }
      mx = warp_max(mx);
      sum = 0.f;
#pragma unroll
      for (int k = 0; k < KJ; k++) {
        const int j = lane + 32 * k;
        g[k] = j < N ? exp2f(g[k] - mx) : 0.f;
        sum += g[k];
      }
      rsum = 1.f / warp_sum(sum);
#pragma unroll
      for (int k = 0; k < KJ; k++) {
        const int j = lane + 32 * k;
        if (j < N) wr[N + j] = g[k] * rsum;
      }
      __syncwarp();
      // pattern row i (lanes over t), P^ s_r = (P - mr) (rr s_r = 1), and its gradient terms
      float cs[32], ct[32];
#pragma unroll
      for (int m = 0; m < 32; m++) cs[m] = ct[m] = 0.f;
      for (int t = lane; t < S; t += 32) {
        float ps = 0.f, pt = 0.f;
        for (int j = 0; j < N; j++) {
          const float xv = xr[j * rs + t];
          ps = fmaf(wr[j], xv, ps);
          pt = fmaf(wr[N + j], xv, pt);
        }
        ps -= mr;
        pt -= mr;
#pragma unroll
        for (int m = 0; m < 32; m++) {
          if (m < M) {
            const float gy = dYs[m * S + t];
            cs[m] = fmaf(gy, ps, cs[m]);
            ct[m] = fmaf(gy, pt, ct[m]);
          }
        }
      }
#pragma unroll
      for (int m = 0; m < 32; m++) {
        if (m < M) {
          const float vs = warp_sum(cs[m]), vt = warp_sum(ct[m]);
          if (lane == 0) {
            acc[m * N + i] += vs;
            acc[(M + m) * N + i] += vt;
          }
        }
      }
      __syncwarp();
    }
    for (int k = threadIdx.x; k < H; k += blockDim.x) accB[k] = fmaf(dYs[k], sr, accB[k]);
  }
  __syncthreads();
  const int E = 2 * M * N + H;
  float* out = part + ((int64_t)c * gridDim.x + blockIdx.x) * E;
  for (int e = threadIdx.x; e < E; e += blockDim.x) out[e] = e < 2 * M * N ? acc[e] : accB[e - 2 * M * N];
}

}  // namespace

bool plan_bwd_head(const FwdArgs& a, int max_smem_optin, BwdPlan* p) {
  if (a.N < 1 || a.M > 32) return false;
  p->mma_mode = false;
  // the tensor-core kernel where it applies (PRNET_BWD_F32=1: this file's FP32 kernel, A/B)
  static const bool force_f32 = [] {
    const char* e = getenv("PRNET_BWD_F32");
    return e && atoi(e) != 0;
  }();
  if (!force_f32 && plan_bwd_head_mma(a, max_smem_optin, p)) return true;
  if (a.N > 32 || a.S > 128) {   // long mode (prnet_bwd_long_kernel)
    if (a.N > 512) return false;
    p->long_mode = true;
    p->ly.np = a.N <= 64 ? 2 : (a.N <= 128 ? 4 : (a.N <= 256 ? 8 : 16));   // KJ
    p->ly.mp = a.S | 1;                                                     // row stride
    p->warps = 8;
    const size_t floats = (size_t)2 * a.N * p->ly.mp + 3 * a.N + 64 + (size_t)p->warps * 2 * a.N +
                          (size_t)a.M * a.S + 2 * (size_t)a.M * a.N + a.H;
    p->smem_bytes = floats * 4;
    if (p->smem_bytes > (size_t)max_smem_optin) return false;
    p->ly.wins_per_cta = 16;
    p->nblk = (int)((a.B + p->ly.wins_per_cta - 1) / p->ly.wins_per_cta);
    p->elems = 2 * a.M * a.N + a.H;
    return true;
  }
  p->long_mode = false;
  BwdLayout& ly = p->ly;
  ly.np = a.N <= 8 ? 8 : (a.N <= 16 ? 16 : 32);
  ly.mp = a.M <= 8 ? 8 : (a.M <= 16 ? 16 : 32);
  const int xz = std::max(2 * a.S * ly.np, 2 * a.M * 32);
  ly.off_dy = (xz + 3) & ~3;
  ly.off_db = (ly.off_dy + a.S * ly.mp + 3) & ~3;
  ly.per_warp = (ly.off_db + a.H + 3) & ~3;
  int w = 12;
  while (w > 1 && (size_t)w * ly.per_warp * 4 > (size_t)max_smem_optin) w--;
  if ((size_t)w * ly.per_warp * 4 > (size_t)max_smem_optin) return false;
  p->warps = w;
  ly.wins_per_cta = 256;   // ~21 series per warp at 12 warps
  p->nblk = (int)((a.B + ly.wins_per_cta - 1) / ly.wins_per_cta);
  p->smem_bytes = (size_t)w * ly.per_warp * 4;
  p->elems = 2 * a.M * a.N + a.H;
  return true;
}

template <int NP, int MP>
static cudaError_t launch_bwd_t(const FwdArgs& a, const BwdPlan& p, const float* dy,
                                float* part, cudaStream_t st) {
  auto k = prnet_bwd_head_kernel<NP, MP>;
  cudaError_t e =
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)p.nblk, (unsigned)a.C);
  k<<<grid, 32 * p.warps, p.smem_bytes, st>>>(a, dy, part, p.ly);
  return cudaGetLastError();
}
template <int NP>
static cudaError_t launch_bwd_n(const FwdArgs& a, const BwdPlan& p, const float* dy,
                                float* part, cudaStream_t st) {
  switch (p.ly.mp) {
    case 8: return launch_bwd_t<NP, 8>(a, p, dy, part, st);
    case 16: return launch_bwd_t<NP, 16>(a, p, dy, part, st);
    default: return launch_bwd_t<NP, 32>(a, p, dy, part, st);
  }
}

cudaError_t launch_bwd_head(const FwdArgs& a, const BwdPlan& p, const float* dy, float* part,
                            float* dws, float* dwt, float* db, int Cw, cudaStream_t st) {
  if (p.nblk > 0 && p.mma_mode) {
    cudaError_t e = launch_bwd_head_mma(a, p, dy, part, st);
    if (e != cudaSuccess) return e;
  } else if (p.nblk > 0 && p.long_mode) {
    cudaError_t e;
    auto go = [&](auto kern) {
      cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)p.smem_bytes);
      if (r != cudaSuccess) return r;
      dim3 grid((unsigned)p.nblk, (unsigned)a.C);
      kern<<<grid, 32 * p.warps, p.smem_bytes, st>>>(a, dy, part, p.ly.mp, p.ly.wins_per_cta);
      return cudaGetLastError();
    };
    switch (p.ly.np) {
      case 2: e = go(prnet_bwd_long_kernel<2>); break;
      case 4: e = go(prnet_bwd_long_kernel<4>); break;
      case 8: e = go(prnet_bwd_long_kernel<8>); break;
      default: e = go(prnet_bwd_long_kernel<16>); break;
    }
    if (e != cudaSuccess) return e;
  } else if (p.nblk > 0) {
    cudaError_t e;
    switch (p.ly.np) {
      case 8: e = launch_bwd_n<8>(a, p, dy, part, st); break;
      case 16: e = launch_bwd_n<16>(a, p, dy, part, st); break;
      default: e = launch_bwd_n<32>(a, p, dy, part, st); break;
    }
    if (e != cudaSuccess) return e;
  }
  dim3 rg((unsigned)((p.elems + 255) / 256), (unsigned)Cw);
  prnet_bwd_reduce_kernel<<<rg, 256, 0, st>>>(part, a.C, p.nblk, p.elems, a.M * a.N, a.H,
                                               a.head_per_channel, dws, dwt, db);
  return cudaGetLastError();
}

}  // namespace prnet
