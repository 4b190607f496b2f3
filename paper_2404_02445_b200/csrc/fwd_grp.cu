// fwd_grp.cu -- "group_f32": the PRNet pattern-attention forward for SHORT series (N <= 16
// segments, S <= 32), FP32 on the CUDA cores, with the lanes of a warp over (series, segment):
// a warp holds G = 32 / NP series at once, NP lanes each (NP = N padded to 2, 4, 8 or 16), lane i
// of a group <-> segment i.  Same reading (SURVEY §8(c) Def 1-11) as every other
// variant; plain FP32, so the arithmetic is warp_f32's.
//
// The short-series stress points are HBM-bound in principle (AI < 11 FLOP/B) but
// the lane-over-time `small_f32` spends ~1280 warp instructions per series on warp-wide
// butterflies.  Here every per-series step is lane-local or a group-local shuffle:
//   a1/a2  lane i loads segment i (S contiguous floats) into registers, descriptors lane-local,
//          sigma^2 by an xor-shuffle tree over the NP lanes of the group;
//   a3     the rows x_j, z_j of the group go to per-warp shared memory; rho_ij from the own z
//          row and broadcast float4 rows (a group reads one address per quarter-warp);
//   a4/a5  both exponentials against the known row maxima (f_i, 0), lane-local row sums;
//   a6/a7  fold: the logits are symmetric, so lane j's row E_j. is column j of E and
//          A[k][j] = E_jk / l_k needs only the row sums of the group (NP shuffles); lane j forms
//          column j of Q = W_s A_s + W_t A_t against W rows broadcast from shared memory;
//   a7/a8  head: lane i takes the future segments m = i, i + NP, ..: Y[m][t] = sum_j Q[m][j]
//          X[j][t] from broadcast rows, + bias, S contiguous floats stored per lane.
#include "prnet_internal.cuh"

namespace prnet {

namespace {

__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }

}  // namespace

// NP: lanes per series (power of two >= N); SQ: float4 chunks per row (S <= 4 SQ)
template <int NP, int SQ>
__global__ void __launch_bounds__(256) prnet_fwd_grp_kernel(FwdArgs a, int wins_per_cta, int mq) {
  constexpr int G = 32 / NP;                 // series per warp
  constexpr int SP = 4 * SQ;
  constexpr int RP = 4 * (SQ | 1);           // row pitch (floats): RP / 4 odd, conflict-free
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int gi = lane / NP, i = lane % NP, gbase = gi * NP;
  const int c = blockIdx.y;
  const int cw = a.head_per_channel ? c : 0;
  const int S = a.S, N = a.N, M = a.M, H = a.H, C = a.C;
  const int QP = NP * mq;                    // Q rows of one group: [M][NP], pitch NP mq (mq odd)

  // ---- CTA: W_s, W_t as [M][NP] (0 past N), bias [H]
  float* wsS = smem;
  float* wtS = wsS + M * NP;
  float* bS = wtS + M * NP;
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
  // ---- per warp: X, Z rows [32][RP], Q of each group [G][M][NP] (pitch QP)
  float* wbase = bS + ((H + 3) & ~3) + warp * (2 * 32 * RP + G * QP);
  float* Xs = wbase;
  float* Zs = Xs + 32 * RP;
  float* Qs = Zs + 32 * RP + gi * QP;
  __syncthreads();

  const bool vec = a.x_vec && (S & 3) == 0;   // 16-byte aligned segment rows
  const bool yvec = (S & 3) == 0 && (H & 3) == 0;
  const float w = a.vtrend;
  const int64_t b_begin = (int64_t)blockIdx.x * wins_per_cta;
  const int64_t b_end = min(b_begin + (int64_t)wins_per_cta, a.B);
  // a1: segment row i of the group's series into registers (Def 2); the next round's row is
  // loaded while this round computes (software pipelining: the DRAM latency of round k + 1
  // overlaps round k's arithmetic instead of stalling every round)
  auto load_row = [&](int64_t bbr, float (&xr)[SP]) {
#pragma unroll
    for (int t = 0; t < SP; t++) xr[t] = 0.f;
    const int64_t br = bbr + gi;
    if (br < b_end && i < N) {
      const float* xg = a.x + br * a.xsb + c * a.xsc + a.r + (int64_t)i * S;
      if (vec) {
#pragma unroll
        for (int q = 0; q < SQ; q++)
          if (4 * q < S) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(xg) + q);
            xr[4 * q] = v.x; xr[4 * q + 1] = v.y; xr[4 * q + 2] = v.z; xr[4 * q + 3] = v.w;
          }
      } else {
#pragma unroll
        for (int t = 0; t < SP; t++)
          if (t < S) xr[t] = __ldg(xg + t);
      }
    }
  };
  // (S <= 16 only: measured, the second row costs S = 24 more occupancy than it hides, L96/S24
  // 0.037 -> 0.046 ms; L96/S12 0.057 -> 0.053, L192/S12 0.137 -> 0.127)
  constexpr bool PF = SP <= 16;
  const int64_t bstep = (int64_t)nwarps * G;
  float xnext[SP];
  if constexpr (PF) load_row(b_begin + (int64_t)warp * G, xnext);
  for (int64_t bb = b_begin + (int64_t)warp * G; bb < b_end; bb += bstep) {
    const int64_t b = bb + gi;
    const bool vs = b < b_end;                // this group's series exists
    const bool valid = vs && i < N;
    // ---------------- a1: segment row i (prefetched), then the next round's row
    float x[SP];
    if constexpr (PF) {
#pragma unroll
      for (int t = 0; t < SP; t++) x[t] = xnext[t];
      if (bb + bstep < b_end) load_row(bb + bstep, xnext);
    } else {
      load_row(bb, x);
    }
    // ---------------- a2: descriptors (Def 3-5) from d = x - x0
    const float x0 = x[0];
    float s1 = 0.f, s3 = 0.f;
#pragma unroll
    for (int t = 0; t < SP; t++)
      if (t < S) {
        const float d = x[t] - x0;
        s1 += d;
        s3 = fmaf((float)t - a.half_s, d, s3);
      }
    const float m1 = s1 * a.inv_s;
    const float mu = x0 + m1;
    const float kap = s3 * a.inv_v;
    float z[SP];
    float nu2 = 0.f;
#pragma unroll
    for (int t = 0; t < SP; t++) {
      z[t] = (valid && t < S) ? (x[t] - x0) - m1 : 0.f;
      nu2 = fmaf(z[t], z[t], nu2);
    }
    // sigma^2 over the group about m0 = mu_0 (xor tree inside the NP lanes)
    const float m0 = __shfl_sync(0xffffffffu, mu, gbase);
    const float dd = valid ? mu - m0 : 0.f;
    float sa = dd, sb = valid ? fmaf((float)S * dd, dd, nu2) : 0.f;
#pragma unroll
    for (int o = NP / 2; o > 0; o >>= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
      sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    const float var = fmaf(-(float)S * sa, sa * a.inv_n, sb) * a.inv_ns;
    const float kt = a.kt / (var + kEpsTrend);          // log2(e) / (tau_t (sigma^2 + eps_t))
    const float g = rsqrtf(nu2 + kEpsSeasonal);
    // the seasonal logits are shifted by 1 >= rho_ij (|rho| <= 1), the same for every row, so E
    // stays symmetric (the fold below needs it); the row maximum rho_ii keeps the largest term
    // >= 2^-ks, normal for tau_s >= 1/80 (as tc_quad)
    const float nks = -a.ks;
    // rows of the group -> shared memory
#pragma unroll
    for (int q = 0; q < SQ; q++) {
      *reinterpret_cast<float4*>(Xs + lane * RP + 4 * q) =
          make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
      *reinterpret_cast<float4*>(Zs + lane * RP + 4 * q) =
          make_float4(z[4 * q], z[4 * q + 1], z[4 * q + 2], z[4 * q + 3]);
    }
    __syncwarp();
    // ---------------- a3-a5: rho_ij, Dhat_ij, both exponentials (known row maxima)
    float es[NP], et[NP];
    float ls = 0.f, lt = 0.f;
#pragma unroll
    for (int j = 0; j < NP; j++) {
      const float gj = __shfl_sync(0xffffffffu, g, gbase + j);
      const float muj = __shfl_sync(0xffffffffu, mu, gbase + j);
      const float kj = __shfl_sync(0xffffffffu, kap, gbase + j);
      float G0 = 0.f, G1 = 0.f;
#pragma unroll
      for (int q = 0; q < SQ; q++) {
        const float4 zj = lds4(Zs + (gbase + j) * RP + 4 * q);
        G0 = fmaf(z[4 * q], zj.x, fmaf(z[4 * q + 1], zj.y, G0));
        G1 = fmaf(z[4 * q + 2], zj.z, fmaf(z[4 * q + 3], zj.w, G1));
      }
      const float rho = (G0 + G1) * g * gj;
      const float dm = mu - muj, dk = kap - kj;
      const float D = fmaf(w * dk, dk, dm * dm);
      const bool on = valid && j < N;
      es[j] = on ? fast_ex2(fmaf(rho, a.ks, nks)) : 0.f;   // exponent <= 0
      et[j] = on ? fast_ex2(-D * kt) : 0.f;
      ls += es[j];
      lt += et[j];
    }
    // ---------------- a6/a7: fold, lane j = this lane's index: Q[m][j] = sum_k W_s[m][k]
    // A_s[k][j] + W_t[m][k] A_t[k][j], A[k][j] = E_jk / l_k (symmetric logits)
    const float rs = valid ? 1.f / ls : 0.f, rt = valid ? 1.f / lt : 0.f;
#pragma unroll
    for (int k = 0; k < NP; k++) {
      es[k] *= __shfl_sync(0xffffffffu, rs, gbase + k);
      et[k] *= __shfl_sync(0xffffffffu, rt, gbase + k);
    }
    for (int m = 0; m < M; m++) {
      float q = 0.f;
#pragma unroll
      for (int k = 0; k < NP; k += 4) {
        if constexpr (NP >= 4) {
          const float4 ws4 = lds4(wsS + m * NP + k), wt4 = lds4(wtS + m * NP + k);
          q = fmaf(ws4.x, es[k], fmaf(ws4.y, es[k + 1], fmaf(ws4.z, es[k + 2], fmaf(ws4.w, es[k + 3], q))));
          q = fmaf(wt4.x, et[k], fmaf(wt4.y, et[k + 1], fmaf(wt4.z, et[k + 2], fmaf(wt4.w, et[k + 3], q))));
        } else {
#pragma unroll
          for (int kk = 0; kk < NP; kk++)
            q = fmaf(wsS[m * NP + kk], es[kk], fmaf(wtS[m * NP + kk], et[kk], q));
        }
      }
      Qs[m * NP + i] = q;
    }
    __syncwarp();
    // ---------------- a7/a8: head Y[m][.] = sum_j Q[m][j] X[j][.], m = i, i + NP, ..; + bias
    if (vs) {
      float* yg = a.y + (b * C + c) * (int64_t)H;
      for (int m = i; m < M; m += NP) {
        float y[SP];
#pragma unroll
        for (int t = 0; t < SP; t++) y[t] = 0.f;
#pragma unroll
        for (int j = 0; j < NP; j++) {
          if (j >= N) break;
          const float qj = Qs[m * NP + j];
#pragma unroll
          for (int q = 0; q < SQ; q++) {
            const float4 xj = lds4(Xs + (gbase + j) * RP + 4 * q);
            y[4 * q] = fmaf(qj, xj.x, y[4 * q]);
            y[4 * q + 1] = fmaf(qj, xj.y, y[4 * q + 1]);
            y[4 * q + 2] = fmaf(qj, xj.z, y[4 * q + 2]);
            y[4 * q + 3] = fmaf(qj, xj.w, y[4 * q + 3]);
          }
        }
        const int h0 = m * S;
        if (yvec) {   // S % 4 == 0, H % 4 == 0: whole float4 chunks inside or outside H
#pragma unroll
          for (int q = 0; q < SQ; q++)
            if (4 * q < S && h0 + 4 * q < H) {
              const float4 bv = lds4(bS + h0 + 4 * q);
              stg_stream4(yg + h0 + 4 * q, make_float4(y[4 * q] + bv.x, y[4 * q + 1] + bv.y,
                                                       y[4 * q + 2] + bv.z, y[4 * q + 3] + bv.w));
            }
        } else {
#pragma unroll
          for (int t = 0; t < SP; t++)
            if (t < S && h0 + t < H) yg[h0 + t] = y[t] + bS[h0 + t];
        }
      }
    }
    __syncwarp();   // the rows and Q are rewritten next round
  }
}

bool plan_grp_kernel(const FwdArgs& a, int max_smem_optin, GrpPlan* p) {
  if (a.N < 1 || a.N > 16 || a.S > 32 || a.S < 2) return false;
  p->np = a.N <= 2 ? 2 : (a.N <= 4 ? 4 : (a.N <= 8 ? 8 : 16));
  p->sq = (a.S + 3) / 4;
  p->mq = a.M | 1;
  const int RP = 4 * (p->sq | 1), G = 32 / p->np;
  const size_t cta = (size_t)(2 * a.M * p->np + ((a.H + 3) & ~3)) * 4;
  const size_t per_warp = (size_t)(2 * 32 * RP + G * p->np * p->mq) * 4;
  int w = 8;
  while (w > 1 && cta + w * per_warp > (size_t)max_smem_optin) w--;
  if (cta + w * per_warp > (size_t)max_smem_optin) return false;
  p->warps = w;
  p->smem_bytes = cta + w * per_warp;
  p->wins_per_cta = w * G * 4;   // 4 rounds per warp
  return true;
}

template <int NP, int SQ>
static cudaError_t launch_grp_t(const FwdArgs& a, const GrpPlan& p, cudaStream_t st) {
  auto k = prnet_fwd_grp_kernel<NP, SQ>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((a.B + p.wins_per_cta - 1) / p.wins_per_cta), (unsigned)a.C);
  k<<<grid, 32 * p.warps, p.smem_bytes, st>>>(a, p.wins_per_cta, p.mq);
  return cudaGetLastError();
}

template <int NP>
static cudaError_t launch_grp_n(const FwdArgs& a, const GrpPlan& p, cudaStream_t st) {
  switch (p.sq) {
    case 1: return launch_grp_t<NP, 1>(a, p, st);
    case 2: return launch_grp_t<NP, 2>(a, p, st);
    case 3: return launch_grp_t<NP, 3>(a, p, st);
    case 4: return launch_grp_t<NP, 4>(a, p, st);
    case 5: return launch_grp_t<NP, 5>(a, p, st);
    case 6: return launch_grp_t<NP, 6>(a, p, st);
    case 7: return launch_grp_t<NP, 7>(a, p, st);
    default: return launch_grp_t<NP, 8>(a, p, st);
  }
}

cudaError_t launch_grp_kernel(const FwdArgs& a, const GrpPlan& p, cudaStream_t st) {
  switch (p.np) {
    case 2: return launch_grp_n<2>(a, p, st);
    case 4: return launch_grp_n<4>(a, p, st);
    case 8: return launch_grp_n<8>(a, p, st);
    default: return launch_grp_n<16>(a, p, st);
  }
}

}  // namespace prnet
