// fwd_small.cu -- fused PRNet pattern-attention forward for SHORT series (N <= 16 segments,
// S <= 128): "small_f32" variant, FP32 throughout (the warp_f32 arithmetic), with the
// lanes of a warp over TIME instead of over segments.
//
// With N <= 8 a lane-per-segment layout (warp_f32, mma_f16x3) leaves 24..31 lanes idle and
// walks S serially; here one warp owns one (window, channel) series, lane l holds the
// values t = l, l + 32, .. of every segment (coalesced loads of each segment row), and the
// few per-series reductions (segment sums, Gram entries) are warp butterflies that leave
// one reduced value per lane (reduce-scatter: 31 shuffles for 32 values) in shared memory.
// The N x N attention is computed element-per-lane (e = i NP + j), its rows reduced with
// xor shuffles inside NP-lane groups; fold Q = W_s A_s + W_t A_t element-per-lane from
// shared memory; the head Y = Q X and the store run lane-over-time again (coalesced).
//
// Same reading (SURVEY §8(c) Def 1-11) and step map as fwd_warp.cu:
//   a1 segment rows x[r + n S + t]; a2 descriptors from d = x - x0 (exact zeros for a
//   constant segment); a3 rho = <z_i, z_j> inv_i inv_j; a4 Dhat; a5 two row softmaxes
//   with the known row maxima (f_i for the seasonal branch, 0 for the trend); a6+a7 fold
//   and head; a8 y = Y + b.  nu2_n is the Gram diagonal G_nn.
#include "prnet_internal.cuh"

namespace prnet {

namespace {

// Reduce P (power of two, <= 32) per-lane partials across the warp; afterwards lane l
// holds in v[0] the total of index l >> (5 - log2 P) (butterfly reduce-scatter: at xor
// offset O the lanes with bit O set keep the upper half of the CNT live values).
template <int CNT, int O, int P>
__device__ __forceinline__ void reduce_scatter_step(float (&v)[P], int lane) {
  if constexpr (O >= 1) {
    if constexpr (CNT > 1) {
      const bool up = (lane & O) != 0;
#pragma unroll
      for (int k = 0; k < CNT / 2; k++) {
        const float send = up ? v[k] : v[k + CNT / 2];
        const float keep = up ? v[k + CNT / 2] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, O);
      }
      reduce_scatter_step<CNT / 2, O / 2, P>(v, lane);
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], O);
      reduce_scatter_step<1, O / 2, P>(v, lane);
    }
  }
}
template <int P>
__device__ __forceinline__ float warp_reduce_scatter(float (&v)[P], int lane) {
  reduce_scatter_step<P, 16, P>(v, lane);
  return v[0];
}
template <int P>
__host__ __device__ constexpr int log2c() { return P <= 1 ? 0 : 1 + log2c<P / 2>(); }

// write the P totals to out[0..P): one lane per index
template <int P>
__device__ __forceinline__ void warp_reduce_to(float (&v)[P], float* out, int lane) {
  const float r = warp_reduce_scatter<P>(v, lane);
  constexpr int sh = 5 - log2c<P>();
  if ((lane & ((1 << sh) - 1)) == 0) out[lane >> sh] = r;
}

// MUFU reciprocal / square root (approximate, <= ~1 ulp) for the per-series scalars and the
// row-sum reciprocals: the IEEE sequences (slow-path branches) were ~20 % of this issue-bound
// kernel's instructions
__device__ __forceinline__ float rcp_a(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float sqrt_a(float v) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

}  // namespace

// NP: padded segment count (power of two >= N, <= 8); TS: time slots per lane (S <= 32 TS)
// Gram partial sums for the pairs e in [LO, LO + P) (e = i NP - i (i - 1) / 2 + j - i, i <= j),
// reduced across the warp into red[LO..LO + P)
template <int NP, int TS, int LO, int P>
__device__ __forceinline__ void gram_batch(const float (&zv)[NP][TS], float* red, int lane) {
  float g[P];
#pragma unroll
  for (int q = 0; q < P; q++) g[q] = 0.f;
#pragma unroll
  for (int i = 0; i < NP; i++)
#pragma unroll
    for (int j = 0; j < NP; j++) {
      if (j < i) continue;
      const int e = i * NP - i * (i - 1) / 2 + (j - i);   // compile-time after unrolling
      if (e < LO || e >= LO + P) continue;
      float sacc = 0.f;
#pragma unroll
      for (int k = 0; k < TS; k++) sacc = fmaf(zv[i][k], zv[j][k], sacc);
      g[e - LO] = sacc;
    }
  warp_reduce_to<P>(g, red + LO, lane);
}
template <int NP, int TS, int LO>
__device__ __forceinline__ void gram_all(const float (&zv)[NP][TS], float* red, int lane) {
  constexpr int NG = NP * (NP + 1) / 2;
  if constexpr (LO < NG) {
    constexpr int R = NG - LO;
    constexpr int P = R >= 32 ? 32 : (R > 8 ? 16 : (R > 4 ? 8 : (R > 2 ? 4 : 2)));
    gram_batch<NP, TS, LO, P>(zv, red, lane);
    gram_all<NP, TS, LO + P>(zv, red, lane);
  }
}

template <int NP, int TS>
__global__ void __launch_bounds__(256) prnet_fwd_small_kernel(FwdArgs a, int wins_per_cta) {
  constexpr int NG = NP * (NP + 1) / 2;                      // Gram entries i <= j
  constexpr int RED = (NG + 31) / 32 * 32 + 32;               // reduced sums (+ slack)
  constexpr int PD = 2 * NP;                                  // s1, s3 per segment
  constexpr int NE = (NP * NP + 31) / 32;                     // attention elements per lane
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int c = blockIdx.y;
  const int cw = a.head_per_channel ? c : 0;
  const int S = a.S, N = a.N, M = a.M, H = a.H, C = a.C;

  // ---- CTA-shared head of channel c: W_s, W_t as [M][NP] (zeros past N), bias [H]
  float* wsS = smem;
  float* wtS = wsS + 32 * NP;
  float* bS = wtS + 32 * NP;
  {
    const float* gws = a.ws + (int64_t)cw * M * N;
    const float* gwt = a.wt + (int64_t)cw * M * N;
    for (int k = threadIdx.x; k < M * NP; k += blockDim.x) {
      const int m = k / NP, n = k - m * NP;
      wsS[k] = n < N ? __ldg(gws + m * N + n) : 0.f;
      wtS[k] = n < N ? __ldg(gwt + m * N + n) : 0.f;
    }
    const float* gb = a.bias + (int64_t)cw * H;
    for (int k = threadIdx.x; k < H; k += blockDim.x) bS[k] = __ldg(gb + k);
  }
  __syncthreads();
  // per-warp scratch: reduced sums [RED], mu / kappa table [2 NP], A_s, A_t [NP][NP],
  // Q [M][NP]
  float* red = bS + ((a.H + 3) & ~3) + warp * (RED + 2 * NP + 2 * NP * NP + 32 * NP);
  float* dtab = red + RED;
  float* as_ = dtab + 2 * NP;
  float* at_ = as_ + NP * NP;
  float* qs = at_ + NP * NP;

  const float sq_vtrend = sqrtf(a.vtrend);   // once, outside the series loop
  const int64_t b_begin = (int64_t)blockIdx.x * wins_per_cta;
  int64_t b_end = b_begin + wins_per_cta;
  if (b_end > a.B) b_end = a.B;
  for (int64_t b = b_begin + warp; b < b_end; b += nwarps) {
    // ---------------- a1: segment rows, lane over time (Def 2)
    const float* xg = a.x + b * a.xsb + c * a.xsc + a.r;
    float xv[NP][TS];
#pragma unroll
    for (int n = 0; n < NP; n++)
#pragma unroll
      for (int k = 0; k < TS; k++) {
        const int t = lane + 32 * k;
        xv[n][k] = (n < N && t < S) ? __ldg(xg + n * S + t) : 0.f;
      }
    // ---------------- a2: descriptors (Def 4) from d = x - x0
    float x0[NP], dsum[PD];
#pragma unroll
    for (int n = 0; n < NP; n++) {
      x0[n] = __shfl_sync(0xffffffffu, xv[n][0], 0);
      float s1 = 0.f, s3 = 0.f;
#pragma unroll
      for (int k = 0; k < TS; k++) {
        const int t = lane + 32 * k;
        const float d = t < S ? xv[n][k] - x0[n] : 0.f;
        xv[n][k] = d;                       // keep d
        s1 += d;
        s3 = fmaf((float)t - a.half_s, d, s3);
      }
      dsum[n] = s1;
      dsum[NP + n] = s3;
    }
    warp_reduce_to<PD>(dsum, red, lane);
    __syncwarp();
    float m1[NP];
#pragma unroll
    for (int n = 0; n < NP; n++) m1[n] = red[n] * a.inv_s;
    if (lane == 0) {   // segment means and slopes, read by index below
#pragma unroll
      for (int n = 0; n < NP; n++) {
        dtab[n] = x0[n] + m1[n];
        dtab[NP + n] = red[NP + n] * a.inv_v;
      }
    }
    // z = d - m1 (zero past S), then the Gram entries G_ij = <z_i, z_j> (i <= j)
#pragma unroll
    for (int n = 0; n < NP; n++)
#pragma unroll
      for (int k = 0; k < TS; k++) {
        const int t = lane + 32 * k;
        xv[n][k] = (n < N && t < S) ? xv[n][k] - m1[n] : 0.f;
      }
    __syncwarp();   // red[] (the descriptor sums) was read above
    gram_all<NP, TS, 0>(xv, red, lane);
    __syncwarp();
    auto gram = [&](int i, int j) {   // G_ij, i, j < NP
      const int lo = i < j ? i : j, hi = i < j ? j : i;
      return red[lo * NP - lo * (lo - 1) / 2 + (hi - lo)];
    };
    // ---------------- Def 5: sigma^2 = (1/(N S)) sum_n [nu2_n + S (mu_n - mubar)^2]
    float mbar = 0.f;
#pragma unroll
    for (int n = 0; n < NP; n++) mbar += n < N ? dtab[n] : 0.f;
    mbar *= a.inv_n;
    float var = 0.f;
#pragma unroll
    for (int n = 0; n < NP; n++)
      var += n < N ? gram(n, n) + (float)S * (dtab[n] - mbar) * (dtab[n] - mbar) : 0.f;
    const float inv_var = rcp_a(var * a.inv_ns + kEpsTrend);
    const float cm = sqrt_a(inv_var * a.kt), ck = cm * sq_vtrend;

    // ---------------- a3-a5: attention, element e = i NP + j per lane; known row maxima
#pragma unroll
    for (int q = 0; q < NE; q++) {
      const int e = lane + 32 * q;
      const int i = (e / NP) & (NP - 1), j = e & (NP - 1);
      const bool ok = e < NP * NP && i < N && j < N;
      const float nui = gram(i, i), nuj = gram(j, j);
      const float invi = rsqrtf(nui + kEpsSeasonal), invj = rsqrtf(nuj + kEpsSeasonal);
      const float rho = gram(i, j) * invi * invj;
      const float fi = sqrt_a(nui) * invi;            // rho_ij <= f_i (Cauchy-Schwarz)
      float es = ok ? fast_ex2((rho - fi) * a.ks) : 0.f;
      const float mui = dtab[i], muj = dtab[j], ki = dtab[NP + i], kj = dtab[NP + j];
      const float dm = (mui - muj) * cm, dk = (ki - kj) * ck;
      float et = ok ? fast_ex2(-fmaf(dm, dm, dk * dk)) : 0.f;   // row max 0 at j = i
      float ss = es, st = et;
#pragma unroll
      for (int o = 1; o < NP; o <<= 1) {                        // row sums (NP lanes)
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
        st += __shfl_xor_sync(0xffffffffu, st, o);
      }
      if (e < NP * NP) {
        as_[e] = ok ? es * rcp_a(ss) : 0.f;   // ss >= its largest term (normal), st >= 1
        at_[e] = ok ? et * rcp_a(st) : 0.f;
      }
    }
    __syncwarp();
    // ---------------- a6+a7 fold Q[m][j] = sum_i W_s[m][i] A_s[i][j] + W_t[m][i] A_t[i][j]
    for (int e = lane; e < M * NP; e += 32) {
      const int m = e / NP, j = e & (NP - 1);
      float acc = 0.f;
#pragma unroll
      for (int i = 0; i < NP; i++)
        acc = fmaf(wsS[m * NP + i], as_[i * NP + j], fmaf(wtS[m * NP + i], at_[i * NP + j], acc));
      qs[e] = acc;
    }
    __syncwarp();
    // ---------------- a7 head Y[m][t] = sum_j Q[m][j] X[j][t] (X = z + mu), a8 store
    float* yg = a.y + (b * C + c) * (int64_t)H;
    for (int m = 0; m < M; m++) {
      float qm[NP], qmu = 0.f;
#pragma unroll
      for (int j = 0; j < NP; j++) {
        qm[j] = qs[m * NP + j];
        qmu = fmaf(qm[j], dtab[j], qmu);
      }
#pragma unroll
      for (int k = 0; k < TS; k++) {
        const int t = lane + 32 * k;
        const int h = m * S + t;
        if (t < S && h < H) {
          float acc = qmu;
#pragma unroll
          for (int j = 0; j < NP; j++) acc = fmaf(qm[j], xv[j][k], acc);
          yg[h] = acc + bS[h];
        }
      }
    }
    __syncwarp();
  }
}

bool plan_small_kernel(const FwdArgs& a, int max_smem_optin, SmallPlan* p) {
  if (a.N > 16 || a.S > 128 || a.M > 32) return false;
  p->np = a.N <= 2 ? 2 : (a.N <= 4 ? 4 : (a.N <= 8 ? 8 : 16));
  p->ts = a.S <= 32 ? 1 : (a.S <= 64 ? 2 : 4);
  p->warps_per_cta = 8;
  const int ng = p->np * (p->np + 1) / 2;
  const int per_warp = (ng + 31) / 32 * 32 + 32 + 2 * p->np + 2 * p->np * p->np + 32 * p->np;
  p->smem_bytes =
      (size_t)(2 * 32 * p->np + ((a.H + 3) & ~3) + p->warps_per_cta * per_warp) * sizeof(float);
  if (p->smem_bytes > (size_t)max_smem_optin) return false;
  p->wins_per_cta = p->warps_per_cta * 4;
  return true;
}

template <int NP, int TS>
static cudaError_t launch_small_t(const FwdArgs& a, const SmallPlan& p, cudaStream_t st) {
  auto k = prnet_fwd_small_kernel<NP, TS>;
  cudaError_t e =
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((a.B + p.wins_per_cta - 1) / p.wins_per_cta), (unsigned)a.C);
  k<<<grid, 32 * p.warps_per_cta, p.smem_bytes, st>>>(a, p.wins_per_cta);
  return cudaGetLastError();
}

template <int NP>
static cudaError_t launch_small_n(const FwdArgs& a, const SmallPlan& p, cudaStream_t st) {
  switch (p.ts) {
    case 1: return launch_small_t<NP, 1>(a, p, st);
    case 2: return launch_small_t<NP, 2>(a, p, st);
    default: return launch_small_t<NP, 4>(a, p, st);
  }
}

cudaError_t launch_small_kernel(const FwdArgs& a, const SmallPlan& p, cudaStream_t st) {
  switch (p.np) {
    case 2: return launch_small_n<2>(a, p, st);
    case 4: return launch_small_n<4>(a, p, st);
    case 8: return launch_small_n<8>(a, p, st);
    default: return launch_small_n<16>(a, p, st);
  }
}

}  // namespace prnet
