// fwd_lane.cu -- "lane_f32": the PRNet pattern-attention forward for FEW-SEGMENT series
// (N <= 8, S % 4 == 0, L = N S <= 192), FP32 on the CUDA cores, ONE LANE PER SERIES.
//
// With N <= 8 the per-series arithmetic is small (N (N + 1) / 2 S Gram FMAs, 2 N^2
// exponentials, the fold and the head) and the stress points that have it are HBM-bound in
// principle (AI < 11 FLOP/B).  The lane-over-segment kernels (group_f32,
// small_f32) spend their time moving rows between lanes (shared-memory broadcasts, warp
// butterflies: 280 warp instructions and ~290 shared wavefronts per series at L96/S12).  Here a
// lane owns a whole series and never talks to another lane:
//   * a warp takes a ROUND of 32 consecutive windows of one channel (lane l <- window 32 r + l),
//     so the channel head W_s, W_t, b is warp-uniform (broadcast loads);
//   * the 32 lookback rows of the next round are fetched while this round computes: the warp
//     copies them row after row with coalesced cp.async (16 bytes per lane; 4 for unaligned
//     sliding windows) into a double-buffered per-warp staging tile, one commit group per round;
//   * rows sit in shared memory with a pitch of an odd number of 16-byte units, so the 32
//     lanes' 128-bit reads of "their" rows at the same offset are conflict-free: every pass
//     (descriptors, Gram, head) re-reads the row at full shared-memory bandwidth;
//   * Gram, logits, both softmaxes (the seasonal one against the exact row maximum, so every
//     tau_s > 0), the fold and the head are lane-local FP32 (the warp_f32 arithmetic);
//   * y leaves through shared memory: every MR head rows (MR S contiguous floats of y) are staged
//     in the lane's output row and the warp writes the 32 staged rows one after another as
//     coalesced 16-byte streaming stores.
// Grid: persistent, CTAs of `warps` warps, rounds dealt round-robin over all warps.
//
// Same reading (SURVEY §8(c) Def 1-11) as every other variant:
//   a1 segment rows x[r + n S + t]; a2 descriptors from d = x - x0 (Def 3-5); a3 rho_ij =
//   <z_i, z_j> g_i g_j, g = (nu2 + eps_s)^(-1/2) (Def 6); a4 Dhat (Def 7); a5 row softmaxes
//   (Def 8); a6+a7 fold Q = W_s A_s + W_t A_t and head Y = Q X (Def 9-10); a8 y = Y + b (Def 11).
#include "prnet_internal.cuh"
#include "mma_common.cuh"

namespace prnet {

namespace {

__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void stg_cs4(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

}  // namespace

// NC: the segment count N (1..8, compile time); MR: head rows per pass (registers)
template <int NC, int MR>
__global__ void __launch_bounds__(256, 1) prnet_fwd_lane_kernel(FwdArgs a, int rounds_per_channel,
                                                                int px, int po) {
  constexpr int N = NC;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int S = a.S, M = a.M, H = a.H, C = a.C;
  const int S4 = S >> 2;
  float* stage = reinterpret_cast<float*>(smem) + (size_t)warp * 32 * (2 * px + po);
  float* outs = stage + 2 * 32 * px;   // output staging: row l = lane l's next MR head rows

  const int64_t items = (int64_t)C * rounds_per_channel;
  const int64_t gw = (int64_t)blockIdx.x * nwarps + warp;
  const int64_t nw = (int64_t)gridDim.x * nwarps;
  // the 32 rows of a round are fetched by the whole warp, row after row, as coalesced cp.async
  // (16 bytes per lane when every row start is 16-byte aligned, else 4), into the aligned
  // staging rows; one commit group per round, two staging buffers
  const bool vec = a.x_vec != 0;
  const int NS = N * S;
  auto issue = [&](int64_t item, int buf) {
    const int c = (int)(item / rounds_per_channel);
    const int64_t b0 = (item - (int64_t)c * rounds_per_channel) * 32;
    const int nrow = (int)min((int64_t)32, a.B - b0);
    float* dst = stage + (size_t)buf * 32 * px;
    const float* src = a.x + b0 * a.xsb + c * a.xsc + a.r;
    if (vec) {
      const int ns4 = NS >> 2;
      for (int l = 0; l < nrow; l++, dst += px, src += a.xsb)
        for (int q = lane; q < ns4; q += 32) cp_async16(dst + 4 * q, src + 4 * q);
    } else {
      for (int l = 0; l < nrow; l++, dst += px, src += a.xsb)
        for (int t = lane; t < NS; t += 32) cp_async4(dst + t, src + t);
    }
    cp_async_commit();
  };

  if (gw < items) issue(gw, 0);
  uint32_t k = 0;
  for (int64_t item = gw; item < items; item += nw, k++) {
    const int buf = k & 1;
    const bool more = item + nw < items;
    if (more) issue(item + nw, buf ^ 1);   // read in round k - 1 (synced below)
    const int c = (int)(item / rounds_per_channel);
    const int cw = a.head_per_channel ? c : 0;
    const int64_t b0 = (item - (int64_t)c * rounds_per_channel) * 32;
    const int nrow = (int)min((int64_t)32, a.B - b0);
    if (more) asm volatile("cp.async.wait_group 1;" ::: "memory");   // round k's group
    else cp_async_wait_all();
    __syncwarp();
    {   // every lane computes (idle lanes of a short round on stale rows, never stored)
      const float* xr = stage + (size_t)buf * 32 * px + lane * px;
      // ---------------- a1+a2: descriptors (Def 3-5) from d = x - x0
      float x0[N], m1[N], mu[N], kap[N];
#pragma unroll
      for (int n = 0; n < N; n++) {
        x0[n] = lds4(xr + n * S).x;   // (a 16-byte read: conflict-free across the lanes)
        float s1a = 0.f, s1b = 0.f, s3a = 0.f, s3b = 0.f;
        for (int q = 0; q < S4; q++) {
          const float4 v = lds4(xr + n * S + 4 * q);
          const float t0 = (float)(4 * q) - a.half_s;
          const float d0 = v.x - x0[n], d1 = v.y - x0[n], d2 = v.z - x0[n], d3 = v.w - x0[n];
          s1a += d0 + d1;
          s1b += d2 + d3;
          s3a = fmaf(t0, d0, fmaf(t0 + 1.f, d1, s3a));
          s3b = fmaf(t0 + 2.f, d2, fmaf(t0 + 3.f, d3, s3b));
        }
        m1[n] = (s1a + s1b) * a.inv_s;
        mu[n] = x0[n] + m1[n];
        kap[n] = (s3a + s3b) * a.inv_v;
      }
      // ---------------- a3: Gram G_ij = <z_i, z_j>, z = (x - x0) - m1, i <= j
      float G[N][N];
#pragma unroll
      for (int i = 0; i < N; i++)
#pragma unroll
        for (int j = i; j < N; j++) G[i][j] = 0.f;
      for (int q = 0; q < S4; q++) {
        float4 z[N];
#pragma unroll
        for (int n = 0; n < N; n++) {
          const float4 v = lds4(xr + n * S + 4 * q);
          z[n] = make_float4((v.x - x0[n]) - m1[n], (v.y - x0[n]) - m1[n], (v.z - x0[n]) - m1[n],
                             (v.w - x0[n]) - m1[n]);
        }
#pragma unroll
        for (int i = 0; i < N; i++)
#pragma unroll
          for (int j = i; j < N; j++)
            G[i][j] = fmaf(z[i].x, z[j].x, fmaf(z[i].y, z[j].y, fmaf(z[i].z, z[j].z, fmaf(z[i].w, z[j].w, G[i][j]))));
      }
      // Def 5: sigma^2 about m0 = mu_0 (sum_n (mu_n - mubar)^2 = sum d^2 - (sum d)^2 / N)
      float sa = 0.f, sb = 0.f;
#pragma unroll
      for (int n = 0; n < N; n++) {
        const float dd = mu[n] - mu[0];
        sa += dd;
        sb += fmaf((float)S * dd, dd, G[n][n]);
      }
      const float var = fmaf(-(float)S * sa, sa * a.inv_n, sb) * a.inv_ns;
      const float kt = a.kt / (var + kEpsTrend);     // log2(e) / (tau_t (sigma^2 + eps_t))
      // ---------------- a3-a5: logits and both softmaxes; the seasonal row maximum is
      // searched (exact), the trend row maximum is 0 at j = i
      float g[N];
#pragma unroll
      for (int n = 0; n < N; n++) g[n] = rsqrtf(G[n][n] + kEpsSeasonal);
      float As[N][N], At[N][N];
#pragma unroll
      for (int i = 0; i < N; i++) {
        float rmax = -INFINITY;
#pragma unroll
        for (int j = 0; j < N; j++) {
          const float gij = i <= j ? G[i][j] : G[j][i];
          As[i][j] = gij * g[i] * g[j];
          rmax = fmaxf(rmax, As[i][j]);
        }
        const float sh = -rmax * a.ks;
        float ls = 0.f;
#pragma unroll
        for (int j = 0; j < N; j++) {
          As[i][j] = fast_ex2(fmaf(As[i][j], a.ks, sh));
          ls += As[i][j];
        }
        const float rs = 1.f / ls;
#pragma unroll
        for (int j = 0; j < N; j++) As[i][j] *= rs;
      }
#pragma unroll
      for (int i = 0; i < N; i++) {
        At[i][i] = 1.f;
#pragma unroll
        for (int j = i + 1; j < N; j++) {
          const float dm = mu[i] - mu[j], dk = kap[i] - kap[j];
          const float D = fmaf(a.vtrend * dk, dk, dm * dm);
          At[i][j] = At[j][i] = fast_ex2(-D * kt);
        }
      }
#pragma unroll
      for (int i = 0; i < N; i++) {
        float lt = 0.f;
#pragma unroll
        for (int j = 0; j < N; j++) lt += At[i][j];
        const float rt = 1.f / lt;
#pragma unroll
        for (int j = 0; j < N; j++) At[i][j] *= rt;
      }
      // ---------------- a6-a8: per MR head rows: Q[m][j] = sum_i W_s[m][i] A_s[i][j] +
      // W_t[m][i] A_t[i][j] (fold), y[m S + t] = sum_j Q[m][j] x_j[t] + b[m S + t]
      const float* wsg = a.ws + (int64_t)cw * M * N;
      const float* wtg = a.wt + (int64_t)cw * M * N;
      const float* bg = a.bias + (int64_t)cw * H;
      for (int m0 = 0; m0 < M; m0 += MR) {
        float q[MR][N];
#pragma unroll
        for (int r = 0; r < MR; r++) {
          const int m = m0 + r < M ? m0 + r : M - 1;
#pragma unroll
          for (int j = 0; j < N; j++) q[r][j] = 0.f;
#pragma unroll
          for (int i = 0; i < N; i++) {
            const float wsv = __ldg(wsg + m * N + i), wtv = __ldg(wtg + m * N + i);
#pragma unroll
            for (int j = 0; j < N; j++) q[r][j] = fmaf(wsv, As[i][j], fmaf(wtv, At[i][j], q[r][j]));
          }
        }
        // rows m0 .. m0 + MR - 1 of y are contiguous: staged in this lane's output row, then
        // written by the warp row after row as coalesced 16-byte stores
        float* ob = outs + lane * po;
        const int h0 = m0 * S;
        const int nh = min(MR * S, H - h0);
        for (int t4 = 0; t4 < S4; t4++) {
          float4 acc[MR];
#pragma unroll
          for (int r = 0; r < MR; r++) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int j = 0; j < N; j++) {
            const float4 v = lds4(xr + j * S + 4 * t4);
#pragma unroll
            for (int r = 0; r < MR; r++) {
              acc[r].x = fmaf(q[r][j], v.x, acc[r].x);
              acc[r].y = fmaf(q[r][j], v.y, acc[r].y);
              acc[r].z = fmaf(q[r][j], v.z, acc[r].z);
              acc[r].w = fmaf(q[r][j], v.w, acc[r].w);
            }
          }
#pragma unroll
          for (int r = 0; r < MR; r++) {
            const int o = r * S + 4 * t4;
            if (o < nh) {
              const float4 bv = __ldg(reinterpret_cast<const float4*>(bg + h0 + o));
              *reinterpret_cast<float4*>(ob + o) =
                  make_float4(acc[r].x + bv.x, acc[r].y + bv.y, acc[r].z + bv.z, acc[r].w + bv.w);
            }
          }
        }
        __syncwarp();
        {
          const float* orow = outs;
          float* yrow = a.y + ((b0 * C + c) * (int64_t)H + h0);
          for (int l = 0; l < nrow; l++, orow += po, yrow += (int64_t)C * H)
            for (int q = lane; 4 * q < nh; q += 32)
              stg_cs4(yrow + 4 * q, lds4(orow + 4 * q));
        }
        __syncwarp();   // the staging rows are rewritten by the next MR rows
      }
    }
    __syncwarp();   // every lane is done with this buffer before round k + 1 refills it
  }
}

// head rows per pass: MR S <= 96 floats of output staging per lane, MR <= 4 (N <= 4) or 2
static int lane_rows(int N, int S) {
  int mr = 96 / S;
  const int cap = N <= 4 ? 4 : 2;
  if (mr > cap) mr = cap;
  return mr < 1 ? 1 : (mr >= 4 ? 4 : (mr >= 2 ? 2 : 1));
}

bool lane_shape_ok(int N, int S, int H, int L) {
  return N >= 1 && N <= 8 && S >= 4 && (S & 3) == 0 && (H & 3) == 0 && N * S <= 192 && L >= N * S;
}

bool plan_lane_kernel(const FwdArgs& a, int max_smem_optin, int sm_count, LanePlan* p) {
  if (!lane_shape_ok(a.N, a.S, a.H, a.L)) return false;
  const int l4 = (a.N * a.S + 3) / 4;
  p->px = 4 * (l4 | 1);   // row pitch: an odd number of 16-byte units (conflict-free)
  p->mr = lane_rows(a.N, a.S);
  p->po = 4 * ((p->mr * a.S / 4) | 1);
  const size_t per_warp = (size_t)32 * (2 * p->px + p->po) * 4;
  int w = 4;
  while (w > 1 && w * per_warp > (size_t)max_smem_optin / 2) w--;
  p->warps = w;
  p->smem_bytes = w * per_warp;
  if (p->smem_bytes > (size_t)max_smem_optin) return false;
  p->sm_count = sm_count;
  p->rounds_per_channel = (int)((a.B + 31) / 32);
  return true;
}

template <int NC, int MR>
static cudaError_t launch_lane_t(const FwdArgs& a, const LanePlan& p, cudaStream_t st) {
  auto k = prnet_fwd_lane_kernel<NC, MR>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  // persistent grid: every resident CTA slot (registers and shared memory), at most one CTA per
  // `warps` rounds
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32 * p.warps, p.smem_bytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const int64_t items = (int64_t)a.C * p.rounds_per_channel;
  int64_t ctas = (int64_t)p.sm_count * per_sm;
  const int64_t need = (items + p.warps - 1) / p.warps;
  if (need < ctas) ctas = need;
  k<<<(unsigned)(ctas < 1 ? 1 : ctas), 32 * p.warps, p.smem_bytes, st>>>(a, p.rounds_per_channel, p.px,
                                                                        p.po);
  return cudaGetLastError();
}

template <int NC>
static cudaError_t launch_lane_n(const FwdArgs& a, const LanePlan& p, cudaStream_t st) {
  if constexpr (NC <= 4) {
    if (p.mr == 4) return launch_lane_t<NC, 4>(a, p, st);
  }
  if (p.mr == 2) return launch_lane_t<NC, 2>(a, p, st);
  return launch_lane_t<NC, 1>(a, p, st);
}

cudaError_t launch_lane_kernel(const FwdArgs& a, const LanePlan& p, cudaStream_t st) {
  switch (a.N) {
    case 1: return launch_lane_n<1>(a, p, st);
    case 2: return launch_lane_n<2>(a, p, st);
    case 3: return launch_lane_n<3>(a, p, st);
    case 4: return launch_lane_n<4>(a, p, st);
    case 5: return launch_lane_n<5>(a, p, st);
    case 6: return launch_lane_n<6>(a, p, st);
    case 7: return launch_lane_n<7>(a, p, st);
    default: return launch_lane_n<8>(a, p, st);
  }
}

}  // namespace prnet
