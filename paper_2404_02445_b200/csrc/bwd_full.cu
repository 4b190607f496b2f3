// bwd_full.cu -- the full backward pass of the PRNet pattern attention (SURVEY §8(f) f4,
// reading R-f7 in DESIGN.md §3): for an upstream gradient dy = dL/dy, the gradients with
// respect to the input x, the head (W_s, W_t, b) and the temperatures (tau_s, tau_t), for the
// base reading (metric_variant bit 0, the level-only trend, allowed).  Each step is the
// adjoint of one Definition step, applied Def 11 -> Def 2 (the same order and formulas as
// oracle_backward_series, which the GPU tests compare against):
//
//   a8/a7  dY = dy (0 past H); dW_s[m][n] += sum_t dY[m][t] P_s[n][t] (W_t likewise);
//          db += dy; dP_s[n][t] = sum_m W_s[m][n] dY[m][t]
//   a6     dA_s[i][j] = sum_t dP_s[i][t] X[j][t];  dX[j][t] += sum_i A_s[i][j] dP_s[i][t]
//   a5     dl[i][j] = A[i][j] (dA[i][j] - sum_k A[i][k] dA[i][k])
//   a4     dDhat = -dl_t / tau_t, dtau_t += sum dl_t Dhat / tau_t^2, dD = dDhat / (s2 + eps_t),
//          ds2 -= sum dDhat D / (s2 + eps_t)^2, dmu_i = 2 sum_j (mu_i - mu_j)(dD_ij + dD_ji),
//          dkappa_i = 2 w sum_j (kappa_i - kappa_j)(dD_ij + dD_ji)
//   a3     drho = dl_s / tau_s, dtau_s -= sum dl_s rho / tau_s^2,
//          dz_i += g_i sum_j (drho_ij + drho_ji) g_j z_j,
//          dg_i = sum_j (drho_ij + drho_ji) rho_ij / g_i,  dnu2_i = -dg_i g_i^3 / 2
//   a2     ds2: dnu2 += ds2 / (N S), dmu += ds2 2 (mu - mubar) / N;
//          dz += 2 z dnu2 + t~ dkappa / V;  dX += dz + (dmu - sum_t dz) / S
//   a1     dx[r + n S + t] = dX[n][t], dx = 0 on the r dropped points
//
// FP32 on the CUDA cores (a training-side pass, not the timed forward).  Layout: one warp per
// series, lane i = segment i (N <= 32), the rows and the N x N matrices in per-warp shared
// memory (odd row pitches: a lane's own row and a broadcast row are conflict-free); the head
// and bias gradients accumulate per warp over its series in shared memory, the warps are
// reduced in a fixed order into one partial per CTA, and a second kernel sums the partials in
// fp64 in a fixed order (dtau over every channel).  Deterministic, no atomics.
#include <algorithm>

#include "prnet_internal.cuh"

namespace prnet {

namespace {

__device__ __forceinline__ float shfl(float v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

}  // namespace

__global__ void __launch_bounds__(256) prnet_bwd_full_kernel(FwdArgs a, const float* __restrict__ dy,
                                                              float* __restrict__ dx,
                                                              float* __restrict__ part,
                                                              BwdFullLayout ly) {
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int c = blockIdx.y, C = a.C;
  const int cw = a.head_per_channel ? c : 0;
  const int N = a.N, S = a.S, M = a.M, H = a.H, L = a.L, r = a.r;
  const int P = ly.pitch, Q = 33;           // row pitches (odd)
  float* wb = smem + warp * ly.per_warp;
  float* Xs = wb;                           // [32][P] segment rows
  float* Zs = Xs + 32 * P;                  // [32][P] centred rows z
  float* dPs = Zs + 32 * P;                 // [32][P] dP_s, later dz
  float* dPt = dPs + 32 * P;                // [32][P] dP_t
  float* dXs = dPt + 32 * P;                // [32][P] dX
  float* As = dXs + 32 * P;                 // [32][Q] A_s, later drho
  float* At = As + 32 * Q;                  // [32][Q] A_t, later dD
  float* Rh = At + 32 * Q;                  // [32][Q] rho
  float* Dm = Rh + 32 * Q;                  // [32][Q] D (unnormalised)
  float* dYs = Dm + 32 * Q;                 // [M][S]
  float* accW = dYs + M * S;                // [2][M][32] dW_s, dW_t (column = segment)
  float* accB = accW + 2 * M * 32;          // [H]
  float* accT = accB + H;                   // [2] per-lane partials reduced at the end
  const float* Wsg = a.ws + (int64_t)cw * M * N;
  const float* Wtg = a.wt + (int64_t)cw * M * N;

  for (int k = lane; k < 2 * M * 32; k += 32) accW[k] = 0.f;
  for (int k = lane; k < H; k += 32) accB[k] = 0.f;
  float dts = 0.f, dtt = 0.f;               // lane partials of dL/dtau_s, dL/dtau_t
  const int i = lane;
  const bool valid = i < N;
  const float V = 1.0f / a.inv_v;           // S (S^2 - 1) / 12
  const float w = a.vtrend;                 // (S^2 - 1) / 12, 0 for the level-only trend
  const float tau_s = kLog2e / a.ks, tau_t = kLog2e / a.kt;

  const int64_t b0 = (int64_t)blockIdx.x * ly.wins_per_cta;
  const int64_t b1 = min(b0 + (int64_t)ly.wins_per_cta, a.B);
  for (int64_t b = b0 + warp; b < b1; b += nwarps) {
    const int64_t series = b * C + c;
    const float* xg = a.x + b * a.xsb + c * a.xsc + r;
    const float* dyg = dy + series * H;
    // ---------------- forward recompute (Def 2-9), FP32
    for (int k = lane; k < N * S; k += 32) {
      const int n = k / S, t = k - n * S;
      Xs[n * P + t] = __ldg(xg + k);
    }
    for (int k = lane; k < M * S; k += 32) dYs[k] = k < H ? __ldg(dyg + k) : 0.f;
    for (int k = lane; k < H; k += 32) accB[k] += __ldg(dyg + k);
    __syncwarp();
    float mu = 0.f, kap = 0.f, nu2 = 0.f;
    if (valid) {
      const float* xr = Xs + i * P;
      const float x0 = xr[0];
      float s1 = 0.f;
      for (int t = 0; t < S; t++) s1 += xr[t] - x0;
      const float m1 = s1 * a.inv_s;
      mu = x0 + m1;
      float q = 0.f, k3 = 0.f;
      for (int t = 0; t < S; t++) {
        const float z = (xr[t] - x0) - m1;
        Zs[i * P + t] = z;
        q = fmaf(z, z, q);
        k3 = fmaf((float)t - a.half_s, z, k3);
      }
      nu2 = q;
      kap = k3 * a.inv_v;
    }
    __syncwarp();
    // sigma^2 (Def 5) about m0 = mu_0: sum d^2 - (sum d)^2 / N with d = mu - m0
    const float m0 = shfl(mu, 0);
    const float dd = valid ? mu - m0 : 0.f;
    const float sd = warp_sum(dd);
    const float sq = warp_sum(valid ? fmaf((float)S * dd, dd, nu2) : 0.f);
    const float s2 = fmaf(-(float)S * sd, sd * a.inv_n, sq) * a.inv_ns;
    const float den = s2 + kEpsTrend;
    const float mubar = m0 + sd * a.inv_n;
    const float g = rsqrtf(nu2 + kEpsSeasonal);
    // rho row i, D row i, both softmax rows (exact row maxima), stored for the transposes
    float lmax_s = -INFINITY, lmax_t = -INFINITY;
    for (int j = 0; j < N; j++) {
      const float gj = shfl(g, j), muj = shfl(mu, j), kj = shfl(kap, j);   // every lane
      if (valid) {
        float G = 0.f;
        for (int t = 0; t < S; t++) G = fmaf(Zs[i * P + t], Zs[j * P + t], G);
        const float rho = G * g * gj;
        const float dm = mu - muj, dk = kap - kj;
        const float D = fmaf(w * dk, dk, dm * dm);
        Rh[i * Q + j] = rho;
        Dm[i * Q + j] = D;
        lmax_s = fmaxf(lmax_s, rho / tau_s);
        lmax_t = fmaxf(lmax_t, -D / den / tau_t);
      }
    }
    __syncwarp();
    float ls = 0.f, lt = 0.f;
    if (valid) {
      for (int j = 0; j < N; j++) {
        const float es = __expf(Rh[i * Q + j] / tau_s - lmax_s);
        const float et = __expf(-Dm[i * Q + j] / den / tau_t - lmax_t);
        As[i * Q + j] = es;
        At[i * Q + j] = et;
        ls += es;
        lt += et;
      }
      const float ils = 1.f / ls, ilt = 1.f / lt;
      for (int j = 0; j < N; j++) {
        As[i * Q + j] *= ils;
        At[i * Q + j] *= ilt;
      }
    }
    __syncwarp();
    // ---------------- a8/a7: head gradients and dP (lane i owns segment i / column i)
    if (valid) {
      for (int t0 = 0; t0 < S; t0 += 16) {
        const int tn = min(16, S - t0);
        float ps[16], pt[16];
#pragma unroll
        for (int u = 0; u < 16; u++) ps[u] = pt[u] = 0.f;
        for (int j = 0; j < N; j++) {
          const float aj = As[i * Q + j], bj = At[i * Q + j];
#pragma unroll
          for (int u = 0; u < 16; u++)
            if (u < tn) {
              const float xv = Xs[j * P + t0 + u];
              ps[u] = fmaf(aj, xv, ps[u]);
              pt[u] = fmaf(bj, xv, pt[u]);
            }
        }
        for (int m = 0; m < M; m++) {
          float gs = 0.f, gt = 0.f;
#pragma unroll
          for (int u = 0; u < 16; u++)
            if (u < tn) {
              const float dv = dYs[m * S + t0 + u];
              gs = fmaf(dv, ps[u], gs);
              gt = fmaf(dv, pt[u], gt);
            }
          accW[m * 32 + i] += gs;
          accW[(M + m) * 32 + i] += gt;
        }
      }
      for (int t = 0; t < S; t++) {
        float gs = 0.f, gt = 0.f;
        for (int m = 0; m < M; m++) {
          const float dv = dYs[m * S + t];
          gs = fmaf(__ldg(Wsg + m * N + i), dv, gs);
          gt = fmaf(__ldg(Wtg + m * N + i), dv, gt);
        }
        dPs[i * P + t] = gs;
        dPt[i * P + t] = gt;
      }
    }
    __syncwarp();
    // ---------------- a6: dA rows (lane-local) and dX = A^T dP (columns of A)
    float dAs[32], dAt[32];
    if (valid) {
#pragma unroll
      for (int j = 0; j < 32; j++) {
        float vs = 0.f, vt = 0.f;
        if (j < N)
          for (int t = 0; t < S; t++) {
            const float xv = Xs[j * P + t];
            vs = fmaf(dPs[i * P + t], xv, vs);
            vt = fmaf(dPt[i * P + t], xv, vt);
          }
        dAs[j] = vs;
        dAt[j] = vt;
      }
      for (int t = 0; t < S; t++) {
        float v = 0.f;
        for (int k = 0; k < N; k++)
          v = fmaf(As[k * Q + i], dPs[k * P + t], fmaf(At[k * Q + i], dPt[k * P + t], v));
        dXs[i * P + t] = v;
      }
    }
    __syncwarp();
    // ---------------- a5: softmax adjoints -> drho (into As), dD (into At), dtau partials
    const float rref = lmax_s * tau_s;   // the row maximum of rho
    if (valid) {
      float ss = 0.f, st = 0.f;
#pragma unroll
      for (int j = 0; j < 32; j++)
        if (j < N) {
          ss = fmaf(As[i * Q + j], dAs[j], ss);
          st = fmaf(At[i * Q + j], dAt[j], st);
        }
#pragma unroll
      for (int j = 0; j < 32; j++)
        if (j < N) {
          const float dls = As[i * Q + j] * (dAs[j] - ss);
          const float dlt = At[i * Q + j] * (dAt[j] - st);
          const float rho = Rh[i * Q + j], D = Dm[i * Q + j];
          // sum_j dls_ij = 0, so the row reference (its maximum) is subtracted first: the same
          // value, without the cancellation of sum_j dls_ij rho_ij when rho_ij ~ rho_ii
          dts -= dls * (rho - rref) / (tau_s * tau_s);
          const float dDh = -dlt / tau_t;
          dtt += dlt * (D / den) / (tau_t * tau_t);
          dAs[j] = dls / tau_s;     // drho_ij
          dAt[j] = dDh;             // dDhat_ij
        }
    }
    __syncwarp();   // every lane has read its As / At rows
    float ds2 = 0.f;
    if (valid) {
#pragma unroll
      for (int j = 0; j < 32; j++)
        if (j < N) {
          As[i * Q + j] = dAs[j];
          At[i * Q + j] = dAt[j] / den;                       // dD_ij
          ds2 -= dAt[j] * Dm[i * Q + j] / (den * den);
        }
    }
    __syncwarp();
    // ---------------- a4: trend adjoint, dmu / dkappa from dD_ij + dD_ji
    // mu_j, kappa_j of every lane through shuffles (all lanes take part)
    float dmu = 0.f, dkap = 0.f;
    for (int j = 0; j < N; j++) {
      const float muj = shfl(mu, j), kj = shfl(kap, j);   // every lane
      if (valid) {
        const float dsym = At[i * Q + j] + At[j * Q + i];
        dmu = fmaf(2.f * (mu - muj), dsym, dmu);
        dkap = fmaf(2.f * w * (kap - kj), dsym, dkap);
      }
    }
    // ---------------- a3: seasonal adjoint: dz (into dPs), dg -> dnu2
    float dnu2 = 0.f;
    if (valid) {
      float dg = 0.f;
      for (int t = 0; t < S; t++) dPs[i * P + t] = 0.f;
      for (int j = 0; j < N; j++)
        dg = fmaf(As[i * Q + j] + As[j * Q + i], Rh[i * Q + j], dg);
      dg /= g;
      dnu2 = -0.5f * dg * g * g * g;
    }
    for (int j = 0; j < N; j++) {
      const float gj = shfl(g, j);   // every lane
      if (valid) {
        const float cf = (As[i * Q + j] + As[j * Q + i]) * g * gj;
        for (int t = 0; t < S; t++) dPs[i * P + t] = fmaf(cf, Zs[j * P + t], dPs[i * P + t]);
      }
    }
    // ---------------- a2: sigma^2 adjoint, descriptor adjoints, dX
    ds2 = warp_sum(ds2);
    if (valid) {
      dnu2 += ds2 * a.inv_ns;
      dmu += ds2 * 2.f * (mu - mubar) * a.inv_n;
      float sdz = 0.f;
      for (int t = 0; t < S; t++) {
        const float dz = fmaf(2.f * Zs[i * P + t], dnu2,
                              fmaf((float)t - a.half_s, dkap / V, dPs[i * P + t]));
        dPs[i * P + t] = dz;
        sdz += dz;
      }
      const float dmt = (dmu - sdz) * a.inv_s;
      for (int t = 0; t < S; t++) dXs[i * P + t] += dPs[i * P + t] + dmt;
    }
    __syncwarp();
    // ---------------- a1: dx (coalesced), zero on the dropped points
    float* dxg = dx + series * L;
    for (int k = lane; k < r; k += 32) dxg[k] = 0.f;
    for (int k = lane; k < N * S; k += 32) {
      const int n = k / S, t = k - n * S;
      dxg[r + k] = dXs[n * P + t];
    }
    __syncwarp();
  }
  // tau partials of this warp
  dts = warp_sum(dts);
  dtt = warp_sum(dtt);
  if (lane == 0) {
    accT[0] = dts;
    accT[1] = dtt;
  }
  __syncthreads();
  // fixed-order reduction over the warps -> one partial per CTA: [2 M N | H | 2]
  const int E = ly.elems;
  float* pout = part + ((int64_t)c * gridDim.x + blockIdx.x) * E;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    float v = 0.f;
    for (int wv = 0; wv < nwarps; wv++) {
      const float* ob = smem + wv * ly.per_warp;
      const float* aW = ob + 5 * 32 * P + 4 * 32 * Q + M * S;
      if (e < 2 * M * N) {
        const int br = e / (M * N), rem = e - br * M * N, m = rem / N, n = rem - m * N;
        v += aW[(br * M + m) * 32 + n];
      } else if (e < 2 * M * N + H) {
        v += aW[2 * M * 32 + (e - 2 * M * N)];
      } else {
        v += aW[2 * M * 32 + H + (e - 2 * M * N - H)];
      }
    }
    pout[e] = v;
  }
}

// fp64 fixed-order sum of the per-CTA partials: head and bias per head channel, the two
// temperature gradients over every channel (block y == 0 writes them)
__global__ void prnet_bwd_full_reduce_kernel(const float* __restrict__ part, int C, int nblk, int E,
                                             int MN, int H, int hpc, float* dws, float* dwt,
                                             float* db, float* dtau) {
  const int cw = blockIdx.y;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    double v = 0.0;
    const bool tau = e >= 2 * MN + H;
    if (tau && cw != 0) continue;
    const int c0 = (hpc && !tau) ? cw : 0, c1 = (hpc && !tau) ? cw + 1 : C;
    for (int c = c0; c < c1; c++)
      for (int k = 0; k < nblk; k++) v += (double)part[((int64_t)c * nblk + k) * E + e];
    if (e < MN) dws[(int64_t)cw * MN + e] = (float)v;
    else if (e < 2 * MN) dwt[(int64_t)cw * MN + e - MN] = (float)v;
    else if (e < 2 * MN + H) db[(int64_t)cw * H + e - 2 * MN] = (float)v;
    else dtau[e - 2 * MN - H] = (float)v;
  }
}

bool plan_bwd_full(const FwdArgs& a, int max_smem_optin, BwdFullPlan* p) {
  if (a.N < 1 || a.N > 32 || a.M > 64 || a.S > 128) return false;
  BwdFullLayout& ly = p->ly;
  ly.pitch = a.S | 1;
  ly.per_warp = 5 * 32 * ly.pitch + 4 * 32 * 33 + a.M * a.S + 2 * a.M * 32 + a.H + 2;
  ly.per_warp = (ly.per_warp + 3) & ~3;
  int w = 8;
  while (w > 1 && (size_t)w * ly.per_warp * 4 > (size_t)max_smem_optin) w--;
  if ((size_t)w * ly.per_warp * 4 > (size_t)max_smem_optin) return false;
  p->warps = w;
  ly.wins_per_cta = 8 * w;
  p->nblk = (int)((a.B + ly.wins_per_cta - 1) / ly.wins_per_cta);
  ly.elems = 2 * a.M * a.N + a.H + 2;
  p->smem_bytes = (size_t)w * ly.per_warp * 4;
  return true;
}

cudaError_t launch_bwd_full(const FwdArgs& a, const BwdFullPlan& p, const float* dy, float* dx,
                            float* part, float* dws, float* dwt, float* db, float* dtau, int Cw,
                            cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(prnet_bwd_full_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  if (p.nblk > 0) {
    dim3 grid((unsigned)p.nblk, (unsigned)a.C);
    prnet_bwd_full_kernel<<<grid, 32 * p.warps, p.smem_bytes, st>>>(a, dy, dx, part, p.ly);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  const int nb = p.nblk > 0 ? p.nblk : 0;
  dim3 rg((unsigned)((p.ly.elems + 255) / 256), (unsigned)Cw);
  prnet_bwd_full_reduce_kernel<<<rg, 256, 0, st>>>(part, a.C, nb, p.ly.elems, a.M * a.N, a.H,
                                                    a.head_per_channel, dws, dwt, db, dtau);
  return cudaGetLastError();
}

}  // namespace prnet
