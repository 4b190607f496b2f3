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
// FP32 on the CUDA cores (a training-side pass, not the timed forward).  The head gradients
// come from the head-backward kernel (bwd_head.cu, same partial / fixed-order reduce scheme);
// this file computes dx and dtau.  Layout: one warp per series, lane i = segment i (N <= 32),
// the rows (float4 chunks, pitch P with P / 4 odd: a lane's own chunk is conflict-free, other
// rows are broadcasts) and the N x N matrices in per-warp shared memory (the transposes of
// drho and dD go through it), W^T per CTA; the temperature partials are reduced over the warps
// and then over the CTAs in a fixed order (fp64).  Deterministic, no atomics.
#include <algorithm>

#include "prnet_internal.cuh"

namespace prnet {

namespace {

__device__ __forceinline__ float shfl(float v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

}  // namespace

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
// 1/v via MUFU.RCP (approximate, <= 1 ulp; v a normal positive float)
__device__ __forceinline__ float rcp_a(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

// dx and the temperature partials; the head gradients come from the head-backward kernel
// (bwd_head.cu), launched by launch_bwd_full.  Shared memory: the CTA's W_s^T, W_t^T [32][mpad];
// per warp X, dP_s, dP_t, dX [32][P] (P % 4 == 0, P / 4 odd: a lane's own float4 row chunk is
// conflict-free, other rows are broadcasts), A_s, A_t (later drho, dD), rho, D [32][33],
// dY [M][P], mu [32].  Rows and columns past N / S are zero.
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
  const int P = ly.pitch, Q = 33, MP = ly.mpad;
  float* WsT = smem;                        // [32][MP] W_s^T
  float* WtT = WsT + 32 * MP;               // [32][MP] W_t^T
  float* wb = smem + 2 * 32 * MP + warp * ly.per_warp;
  float* Xs = wb;                           // [32][P] segment rows
  float* dPs = Xs + 32 * P;                 // [32][P] dP_s
  float* dPt = dPs + 32 * P;                // [32][P] dP_t
  float* dXs = dPt + 32 * P;                // [32][P] dX (the direct part first)
  float* As = dXs + 32 * P;                 // [32][Q] A_s, then drho
  float* At = As + 32 * Q;                  // [32][Q] A_t, then dD
  float* Rh = At + 32 * Q;                  // [32][Q] rho
  // dY [M][P] lives in the dX buffer between the Gram (its z rows) and the aggregation
  // adjoint (dX), and D_ij is recomputed from (mu_j, kappa_j): 8 warps per SM instead of 6
  float* dYs = dXs;
  float* muv = Rh + 32 * Q;                 // [32] mu_j
  float* gv = muv + 32;                     // [32] g_j = (nu2_j + eps_s)^(-1/2)
  float* x0v = gv + 32;                     // [32] x0_j (z_j = (X_j - x0_j) - m1_j, as Def 4's
  float* m1v = x0v + 32;                    // [32] m1_j  forward: no cancellation against mu)
  float* kv = m1v + 32;                     // [32] kappa_j
  {
    const float* gs = a.ws + (int64_t)cw * M * N;
    const float* gt = a.wt + (int64_t)cw * M * N;
    for (int k = threadIdx.x; k < 32 * MP; k += blockDim.x) {
      const int n = k / MP, m = k - n * MP;
      const bool ok = n < N && m < M;
      WsT[k] = ok ? __ldg(gs + m * N + n) : 0.f;
      WtT[k] = ok ? __ldg(gt + m * N + n) : 0.f;
    }
  }
  for (int k = lane; k < 32 * P; k += 32) Xs[k] = 0.f;   // padding stays 0
  __syncthreads();
  float dts = 0.f, dtt = 0.f;               // lane partials of dL/dtau_s, dL/dtau_t
  const int i = lane;
  const bool valid = i < N;
  const float w = a.vtrend;                 // (S^2 - 1) / 12, 0 for the level-only trend
  const float tau_s = kLog2e / a.ks, tau_t = kLog2e / a.kt;
  const int S4 = (S + 3) >> 2;

  const int64_t b0 = (int64_t)blockIdx.x * ly.wins_per_cta;
  const int64_t b1 = min(b0 + (int64_t)ly.wins_per_cta, a.B);
  // (n, t) of flat index k = lane + 32 u, stepped without an integer division per element
  const int q32 = 32 / S, r32 = 32 - q32 * S;
  const int n_l = lane / S, t_l = lane - n_l * S;
  for (int64_t b = b0 + warp; b < b1; b += nwarps) {
    const int64_t series = b * C + c;
    const float* xg = a.x + b * a.xsb + c * a.xsc + r;
    const float* dyg = dy + series * H;
    for (int k = lane, n = n_l, t = t_l; k < N * S; k += 32) {
      Xs[n * P + t] = __ldg(xg + k);
      n += q32;
      t += r32;
      if (t >= S) { t -= S; n++; }
    }
    __syncwarp();
    // ---------------- forward recompute (Def 3-8), FP32
    float mu = 0.f, kap = 0.f, nu2 = 0.f, x0 = 0.f, m1 = 0.f;
    if (valid) {
      const float* xr = Xs + i * P;
      float* zr = dXs + i * P;   // z rows for the Gram (dXs is first written at a6)
      x0 = xr[0];
      float s1 = 0.f;
      for (int t = 0; t < S; t++) s1 += xr[t] - x0;
      m1 = s1 * a.inv_s;
      mu = x0 + m1;
      float q = 0.f, k3 = 0.f;
      // z (Def 4) formed once into the dX buffer for the Gram below, 0 past S up to the
      // float4 chunk end (the a6 / dz steps keep forming z_j from X_j, exactly as before)
      for (int t = 0; t < S; t++) {
        const float z = (xr[t] - x0) - m1;
        zr[t] = z;
        q = fmaf(z, z, q);
        k3 = fmaf((float)t - a.half_s, z, k3);
      }
      for (int t = S; t < 4 * S4; t++) zr[t] = 0.f;
      nu2 = q;
      kap = k3 * a.inv_v;
    }
    muv[i] = mu;
    kv[i] = kap;
    x0v[i] = x0;
    m1v[i] = m1;
    const float m0 = shfl(mu, 0);
    const float dd = valid ? mu - m0 : 0.f;
    const float sd = warp_sum(dd);
    const float sq = warp_sum(valid ? fmaf((float)S * dd, dd, nu2) : 0.f);
    const float s2 = fmaf(-(float)S * sd, sd * a.inv_n, sq) * a.inv_ns;
    const float den = s2 + kEpsTrend;
    const float mubar = m0 + sd * a.inv_n;
    const float g = rsqrtf(nu2 + kEpsSeasonal);
    gv[i] = g;
    // series-level reciprocals, formed once: the per-element steps below multiply (IEEE
    // divisions inside the N x N loops were 37 % of the kernel's instructions)
    const float its = 1.f / tau_s, itt = 1.f / tau_t, iden = rcp_a(den);
    const float ct = iden * itt;             // Dhat / tau_t = D / (den tau_t)
    __syncwarp();
    // Gram row i: <z_i, z_j> from the own row and broadcast rows (z = X - mu; t >= S masked)
    float lmax_s = -INFINITY, lmax_t = -INFINITY;
    {
      float G[32];
#pragma unroll
      for (int j = 0; j < 32; j++) G[j] = 0.f;
      if (valid)
        for (int q4 = 0; q4 < S4; q4++) {
          const int t0 = 4 * q4;
          const float4 zi = ld4(dXs + i * P + t0);   // z rows, 0 past S
#pragma unroll
          for (int j = 0; j < 32; j++) {
            if (j >= N) break;
            const float4 zj = ld4(dXs + j * P + t0);
            G[j] = fmaf(zi.x, zj.x, fmaf(zi.y, zj.y, fmaf(zi.z, zj.z, fmaf(zi.w, zj.w, G[j]))));
          }
        }
#pragma unroll
      for (int j = 0; j < 32; j++) {
        if (j >= N) break;
        const float gj = shfl(g, j), kj = shfl(kap, j);   // every lane
        if (valid) {
          const float rho = G[j] * g * gj;
          const float dm = mu - muv[j], dk = kap - kj;
          const float D = fmaf(w * dk, dk, dm * dm);
          Rh[i * Q + j] = rho;
          lmax_s = fmaxf(lmax_s, rho * its);
          lmax_t = fmaxf(lmax_t, -D * ct);
        }
      }
    }
    __syncwarp();   // every lane has read the z rows (the Gram): the dX buffer takes dY [M][P]
    for (int m = 0; m < M; m++)
      for (int t = lane; t < P; t += 32) {
        const int h = m * S + t;
        dYs[m * P + t] = (t < S && h < H) ? __ldg(dyg + h) : 0.f;
      }
    __syncwarp();
    if (valid) {
      float ls = 0.f, lt = 0.f;
      for (int j = 0; j < N; j++) {
        const float dm = mu - muv[j], dk = kap - kv[j];
        const float D = fmaf(w * dk, dk, dm * dm);   // as in the Gram loop (same operations)
        const float es = __expf(Rh[i * Q + j] * its - lmax_s);
        const float et = __expf(-D * ct - lmax_t);
        As[i * Q + j] = es;
        At[i * Q + j] = et;
        ls += es;
        lt += et;
      }
      const float ils = rcp_a(ls), ilt = rcp_a(lt);   // row sums >= 1 (the row maximum's term)
      for (int j = 0; j < N; j++) {
        As[i * Q + j] *= ils;
        At[i * Q + j] *= ilt;
      }
      // ---------------- a7: dP_i = W^T[i] dY (W^T row per lane, dY rows broadcast)
      for (int q4 = 0; q4 < S4; q4++) {
        float4 gs = make_float4(0.f, 0.f, 0.f, 0.f), gt = gs;
        for (int m = 0; m < M; m++) {
          const float4 dv = ld4(dYs + m * P + 4 * q4);
          const float ws_ = WsT[i * MP + m], wt_ = WtT[i * MP + m];
          gs.x = fmaf(ws_, dv.x, gs.x); gs.y = fmaf(ws_, dv.y, gs.y);
          gs.z = fmaf(ws_, dv.z, gs.z); gs.w = fmaf(ws_, dv.w, gs.w);
          gt.x = fmaf(wt_, dv.x, gt.x); gt.y = fmaf(wt_, dv.y, gt.y);
          gt.z = fmaf(wt_, dv.z, gt.z); gt.w = fmaf(wt_, dv.w, gt.w);
        }
        st4(dPs + i * P + 4 * q4, gs);
        st4(dPt + i * P + 4 * q4, gt);
      }
    }
    __syncwarp();
    // ---------------- a6: dX_direct = A^T dP (A's columns, dP rows broadcast) and dA rows
    float dAs[32], dAt[32];
#pragma unroll
    for (int j = 0; j < 32; j++) dAs[j] = dAt[j] = 0.f;
    if (valid) {
      for (int q4 = 0; q4 < S4; q4++) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int k = 0; k < N; k++) {
          const float as = As[k * Q + i], at = At[k * Q + i];
          const float4 ps = ld4(dPs + k * P + 4 * q4), pt = ld4(dPt + k * P + 4 * q4);
          v.x = fmaf(as, ps.x, fmaf(at, pt.x, v.x));
          v.y = fmaf(as, ps.y, fmaf(at, pt.y, v.y));
          v.z = fmaf(as, ps.z, fmaf(at, pt.z, v.z));
          v.w = fmaf(as, ps.w, fmaf(at, pt.w, v.w));
        }
        st4(dXs + i * P + 4 * q4, v);
        const float4 ps = ld4(dPs + i * P + 4 * q4), pt = ld4(dPt + i * P + 4 * q4);
#pragma unroll
        for (int j = 0; j < 32; j++) {
          if (j >= N) break;
          const float4 xj = ld4(Xs + j * P + 4 * q4);
          dAs[j] = fmaf(ps.x, xj.x, fmaf(ps.y, xj.y, fmaf(ps.z, xj.z, fmaf(ps.w, xj.w, dAs[j]))));
          dAt[j] = fmaf(pt.x, xj.x, fmaf(pt.y, xj.y, fmaf(pt.z, xj.z, fmaf(pt.w, xj.w, dAt[j]))));
        }
      }
    }
    // ---------------- a5: softmax adjoints (own rows) -> drho, dD, dtau and ds2 partials
    float ds2 = 0.f;
    const float rref = lmax_s * tau_s;   // the row maximum of rho: sum_j dls_ij = 0
    const float its2 = its * its, ctt = ct * itt, iden2 = iden * iden;
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
          const float dm = mu - muv[j], dk = kap - kv[j];
          const float rho = Rh[i * Q + j], D = fmaf(w * dk, dk, dm * dm);
          dts -= dls * (rho - rref) * its2;
          dtt += dlt * D * ctt;      // dlt Dhat / tau_t^2
          const float dDh = -dlt * itt;
          ds2 -= dDh * D * iden2;
          dAs[j] = dls * its;        // drho_ij
          dAt[j] = dDh * iden;       // dD_ij
        }
    }
    __syncwarp();   // every lane has read A's columns (a6) and its own rows
    if (valid) {
#pragma unroll
      for (int j = 0; j < 32; j++)
        if (j < N) {
          As[i * Q + j] = dAs[j];
          At[i * Q + j] = dAt[j];
        }
    }
    __syncwarp();
    // ---------------- a4 / a3 / a2: dmu, dkappa (dD + dD^T), dg (drho + drho^T), ds2
    float dmu = 0.f, dkap = 0.f, dg = 0.f;
#pragma unroll
    for (int j = 0; j < 32; j++) {
      if (j >= N) break;
      const float kj = shfl(kap, j);   // every lane
      if (valid) {
        const float dsym = At[i * Q + j] + At[j * Q + i];
        dmu = fmaf(2.f * (mu - muv[j]), dsym, dmu);
        dkap = fmaf(2.f * w * (kap - kj), dsym, dkap);
        dg = fmaf(As[i * Q + j] + As[j * Q + i], Rh[i * Q + j], dg);
      }
    }
    ds2 = warp_sum(ds2);
    float dnu2 = valid ? -0.5f * dg * g * g : 0.f;   // d(nu2) = -dg g^3 / (2 g) (no division)
    dnu2 += ds2 * a.inv_ns;
    dmu += ds2 * 2.f * (mu - mubar) * a.inv_n;
    // ---------------- dX = dX_direct + dz + dmu / S with dz_i = g_i sum_j (drho_ij + drho_ji)
    // g_j z_j + 2 z_i dnu2 + t~ dkappa / V (sum_t dz_i = 0: every term is centred), -> dx
    float* dxg = dx + series * L;
    for (int k = lane; k < r; k += 32) dxg[k] = 0.f;
    if (valid) {
      float cz[32];
#pragma unroll
      for (int j = 0; j < 32; j++) cz[j] = 0.f;
#pragma unroll
      for (int j = 0; j < 32; j++)
        if (j < N) cz[j] = (As[i * Q + j] + As[j * Q + i]) * g * gv[j];
      for (int q4 = 0; q4 < S4; q4++) {
        const int t0 = 4 * q4;
        float4 v = ld4(dXs + i * P + t0);
        const float4 xi = ld4(Xs + i * P + t0);
        const float dmS = dmu * a.inv_s;
        const float dkv = dkap * a.inv_v;   // 1 / V
        float4 dz;
        dz.x = fmaf(2.f * ((xi.x - x0) - m1), dnu2, ((float)t0 - a.half_s) * dkv);
        dz.y = fmaf(2.f * ((xi.y - x0) - m1), dnu2, ((float)(t0 + 1) - a.half_s) * dkv);
        dz.z = fmaf(2.f * ((xi.z - x0) - m1), dnu2, ((float)(t0 + 2) - a.half_s) * dkv);
        dz.w = fmaf(2.f * ((xi.w - x0) - m1), dnu2, ((float)(t0 + 3) - a.half_s) * dkv);
#pragma unroll
        for (int j = 0; j < 32; j++) {
          if (j >= N) break;
          const float4 xj = ld4(Xs + j * P + t0);
          const float aj = x0v[j], bj = m1v[j], cj = cz[j];
          dz.x = fmaf(cj, (xj.x - aj) - bj, dz.x);
          dz.y = fmaf(cj, (xj.y - aj) - bj, dz.y);
          dz.z = fmaf(cj, (xj.z - aj) - bj, dz.z);
          dz.w = fmaf(cj, (xj.w - aj) - bj, dz.w);
        }
        v.x += dz.x + dmS;
        v.y += dz.y + dmS;
        v.z += dz.z + dmS;
        v.w += dz.w + dmS;
        st4(dXs + i * P + t0, v);
      }
    }
    __syncwarp();
    for (int k = lane, n = n_l, t = t_l; k < N * S; k += 32) {
      dxg[r + k] = dXs[n * P + t];
      n += q32;
      t += r32;
      if (t >= S) { t -= S; n++; }
    }
    __syncwarp();
  }
  dts = warp_sum(dts);
  dtt = warp_sum(dtt);
  float* red = smem + 2 * 32 * MP + nwarps * ly.per_warp;   // [8][2]
  if (lane == 0) {
    red[2 * warp] = dts;
    red[2 * warp + 1] = dtt;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    float v = 0.f;
    for (int wv = 0; wv < nwarps; wv++) v += red[2 * wv + threadIdx.x];
    part[((int64_t)c * gridDim.x + blockIdx.x) * 2 + threadIdx.x] = v;
  }
}
// fp64 fixed-order sum of the per-CTA temperature partials [C][nblk][2] -> dtau[2]
__global__ void prnet_bwd_tau_reduce_kernel(const float* __restrict__ part, int n, float* dtau) {
  const int e = threadIdx.x;
  if (e < 2) {
    double v = 0.0;
    for (int k = 0; k < n; k++) v += (double)part[2 * k + e];
    dtau[e] = (float)v;
  }
}

bool plan_bwd_full(const FwdArgs& a, int max_smem_optin, BwdFullPlan* p) {
  if (a.N < 1 || a.N > 32 || a.M > 32 || a.S > 128) return false;
  if (!plan_bwd_head(a, max_smem_optin, &p->head) || p->head.long_mode) return false;
  BwdFullLayout& ly = p->ly;
  int P = (a.S + 3) & ~3;
  if (((P / 4) & 1) == 0) P += 4;          // P / 4 odd: conflict-free own-row float4 reads
  ly.pitch = P;
  ly.mpad = a.M | 1;                        // odd: W^T row reads by 32 lanes are conflict-free
  ly.per_warp = ((4 * 32 * P + 3 * 32 * 33 + 160) + 3) & ~3;
  const size_t cta = (size_t)2 * 32 * ly.mpad * 4 + 16 * 4;
  int w = 8;
  while (w > 1 && cta + (size_t)w * ly.per_warp * 4 > (size_t)max_smem_optin) w--;
  if (cta + (size_t)w * ly.per_warp * 4 > (size_t)max_smem_optin) return false;
  p->warps = w;
  ly.wins_per_cta = 8 * w;
  p->nblk = (int)((a.B + ly.wins_per_cta - 1) / ly.wins_per_cta);
  ly.elems = 2;
  p->smem_bytes = cta + (size_t)w * ly.per_warp * 4;
  return true;
}

size_t bwd_full_workspace_floats(const FwdArgs& a, const BwdFullPlan& p) {
  return (size_t)a.C * std::max(p.head.nblk, 1) * p.head.elems +
         (size_t)a.C * std::max(p.nblk, 1) * 2;
}

cudaError_t launch_bwd_full(const FwdArgs& a, const BwdFullPlan& p, const float* dy, float* dx,
                            float* work, float* dws, float* dwt, float* db, float* dtau, int Cw,
                            cudaStream_t st) {
  // the head gradients (dW_s, dW_t, db): the head-backward kernel and its fixed-order reduce
  cudaError_t e = launch_bwd_head(a, p.head, dy, work, dws, dwt, db, Cw, st);
  if (e != cudaSuccess) return e;
  float* part = work + (size_t)a.C * std::max(p.head.nblk, 1) * p.head.elems;
  if ((e = cudaFuncSetAttribute(prnet_bwd_full_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)p.smem_bytes)) != cudaSuccess)
    return e;
  if (p.nblk > 0) {
    dim3 grid((unsigned)p.nblk, (unsigned)a.C);
    prnet_bwd_full_kernel<<<grid, 32 * p.warps, p.smem_bytes, st>>>(a, dy, dx, part, p.ly);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  prnet_bwd_tau_reduce_kernel<<<1, 32, 0, st>>>(part, p.nblk > 0 ? a.C * p.nblk : 0, dtau);
  return cudaGetLastError();
}

}  // namespace prnet
