// fwd_mma.cu -- fused PRNet pattern-attention forward on the tensor cores
// (sm_100a mma.sync, split-fp16 "3-product" arithmetic), N <= 32, M <= 32.
//
// Same per-series step map and reading as fwd_warp.cu; what
// changes is how the three contractions run:
//   a3 Gram      G  = Z Z^T            (N x S)(S x N)
//   a6+a7 fold   Q  = W_s A_s + W_t A_t (M x N)(N x N) x 2
//   a7 head      Y  = Q X               (M x N)(N x S)
// each as m16n8k16 (and m16n8k8) MMAs with fp32 accumulation, every fp32
// operand v split into v = hi + lo (both fp16; lo = fp16(v - hi)) and the
// product formed as hi*hi + hi*lo + lo*hi.  The dropped lo*lo term and the
// rounding of lo are ~2^-22 relative, i.e. fp32-class accuracy (
// plain fp16/tf32 fail the 1e-5 + 1e-4|y| bar).  Operands are pre-scaled by
// exact powers of two (per series for X and Z, per channel for W) so fp16
// never overflows; the scales are divided out exactly in fp32.
//
// Data never leaves the SM between load and store: the Gram accumulators are
// softmax-ed in registers (FA2-style quad reductions, packed f32x2 math), the
// attention tiles are transposed in registers with movmatrix into the B
// operand of the fold, and the fold's accumulators are re-packed in registers
// as the A operand of the head.  Shared memory holds only the series (fp32
// staging + fp16 X, Z) and the channel's head (fp16 W, fp32 b).  The next
// series is prefetched with cp.async while the current one is in the tensor
// cores.
//
// Template parameters: MT / MMT = 16-row tiles of segments / future segments;
// SC = compile-time segment length (24: every configs[0..3] shape; dense
// operand rows, lane-per-row register conversion, k16 + k8 Gram) or 0
// (generic runtime S with padded rows); DBG = also dump the attention rows.
#include <cuda_fp16.h>

#include <cmath>

#include "mma_common.cuh"

#ifndef PRNET_MMA_THREADS
#define PRNET_MMA_THREADS 256
#endif
#ifndef PRNET_MMA_MINB
#define PRNET_MMA_MINB 2
#endif

namespace prnet {


// Shared-memory layout, identical on host (plan) and device (compile-time for SC = 24):
// [W' hi | W' lo]  [per-warp regions x nwarps]  [bias fp32 [H]]
// per-warp: xbuf fp32 [nr*S] | X' hi, lo [nr][sph] | Z' hi, lo [nr][zph] | misc (row
// descriptors float4[32], x0/m1/kappa[96], mbarrier, and with `extra` = kCompBytes the
// component-value vectors of the generic path)
struct MmaOffsets {
  int xhi, xlo, zhi, zlo, misc, pw;   // per-warp
  int zhi_bytes;                      // bytes of one Z' plane (Z' hi, lo are contiguous)
  int wlo, wpack;                     // CTA-shared head
};
__host__ __device__ constexpr int r16(int v) { return (v + 15) & ~15; }
// generic path, metric_variant bit 2: [10][32] floats: mu^_s, kappa^_s, A_s mu^_s,
// A_s kappa^_s, A_t mu^_t, A_t kappa^_t, alpha, beta, mu^_t, kappa^_t (the _s and _t inputs
// differ only under the moving-average decomposition)
constexpr int kCompBytes = 10 * 32 * 4;
__host__ __device__ constexpr MmaOffsets mma_offsets(int nr, int S, int sph, int zph, int mmt,
                                                     int extra = 0) {
  MmaOffsets o{};
  int off = r16(nr * S * 4);
  o.xhi = off;
  off = r16(off + nr * sph * 2);
  o.xlo = off;
  off = r16(off + nr * sph * 2);
  o.zhi = off;
  o.zhi_bytes = r16(nr * zph * 2);
  off = r16(off + nr * zph * 2);
  o.zlo = off;
  off = r16(off + nr * zph * 2);
  o.misc = off;
  off += 512 + 384 + 16 + extra;
  o.pw = (off + 127) & ~127;
  const int wph = 2 * nr + 8, rows = 16 * mmt;
  o.wlo = rows * wph * 2;
  o.wpack = r16(2 * rows * wph * 2);
  return o;
}

// DEC: moving-average decomposition (ma_kernel, reading R-f5; generic path only): the
// seasonal branch runs on x - MA(x), the trend branch on MA(x), the head on both
// COMP: the S = 24 instantiation with component values (the generic one has them at run time)
template <int MT, int MMT, int SC, bool DBG, int NC = 0, bool DEC = false, bool COMP = false>
__global__ void __launch_bounds__(PRNET_MMA_THREADS, PRNET_MMA_MINB) prnet_fwd_mma_kernel(FwdArgs a, MmaLayout ly,
                                                               int wins_per_cta) {
  extern __shared__ float4 smem4[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(smem4);
  constexpr int NR = 16 * MT;
  constexpr int WPH = 2 * NR + 8;
  constexpr MmaOffsets KO =
      mma_offsets(NR, SC > 0 ? SC : 8, SC > 0 ? SC : 8, SC > 0 ? SC : 8, MMT, COMP ? kCompBytes : 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int gq = lane >> 2, cq = lane & 3, q8 = lane >> 3;
  const int c = blockIdx.y;
  const int cw = a.head_per_channel ? c : 0;
  const int S = SC > 0 ? SC : a.S;
  // NC > 0: compile-time segment count (30: every L = 720, S = 24 config), so the
  // j < N / i < N masks fold away
  const int N = NC > 0 ? NC : a.N;
  const int M = a.M, H = a.H, C = a.C;
  // operand row strides (halves): dense rows when S is the compile-time 24
  const int sph = SC > 0 ? SC : ly.sph;
  const int zph = SC > 0 ? SC : ly.zph;
  const int ntt = SC > 0 ? (SC + 7) / 8 : ly.ntt;
  const int pw = SC > 0 ? KO.pw : ly.per_warp_bytes;

  // ---------------- CTA-shared: the channel's pre-packed head (prnet_load_params):
  // W' = W * sw as fp16 hi/lo [16*MMT][WPH] (cols: seasonal i at [0, NR), trend i at
  // [NR, 2NR), zeros elsewhere), 1/sw, and the fp32 bias.
  const __half* w_hi = reinterpret_cast<const __half*>(smem);
  const __half* w_lo = reinterpret_cast<const __half*>(smem + KO.wlo);
  float* bS = reinterpret_cast<float*>(smem + KO.wpack + nwarps * pw);
  const float inv_sw = a.wpack_inv_sw[cw];
  {
    const uint4* src = a.wpack + (int64_t)cw * (KO.wpack / 16);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    for (int k = threadIdx.x; k < KO.wpack / 16; k += blockDim.x) dst[k] = __ldg(src + k);
    const float* gb = a.bias + (int64_t)cw * H;
    const int hb = max(H, 16 * MMT * S);   // zero-padded to the epilogue's whole tiles
    for (int k = threadIdx.x; k < hb; k += blockDim.x) bS[k] = k < H ? __ldg(gb + k) : 0.f;
  }

  // ---------------- per-warp: fp32 staging, X' hi/lo [NR][sph], Z' hi/lo [NR][zph]
  unsigned char* wb = smem + KO.wpack + warp * pw;
  float* xbuf = reinterpret_cast<float*>(wb);
  __half* x_hi = reinterpret_cast<__half*>(wb + (SC > 0 ? KO.xhi : ly.off_xhi));
  __half* x_lo = reinterpret_cast<__half*>(wb + (SC > 0 ? KO.xlo : ly.off_xlo));
  __half* z_hi = reinterpret_cast<__half*>(wb + (SC > 0 ? KO.zhi : ly.off_zhi));
  __half* z_lo = reinterpret_cast<__half*>(wb + (SC > 0 ? KO.zlo : ly.off_zlo));
  // per-row descriptors (mu~, kappa~, 1/sqrt(nu2 + eps_s), f) broadcast through shared memory
  float4* dsc = reinterpret_cast<float4*>(wb + (SC > 0 ? KO.misc : ly.off_diag));
  // (the generic path stages its per-row shift / mean / slope / Z' scale in dsc itself)
  float* rsm = reinterpret_cast<float*>(dsc + 32);            // [96] spare
  uint64_t* xbar = reinterpret_cast<uint64_t*>(rsm + 96);     // TMA completion barrier
  float* cvec = rsm + 100;   // generic path, component values: [10][32] (kCompBytes)
  // DEC: fp32 trend of the staged series, trend values X_t' as fp16 hi / lo
  float* tbuf = DEC ? reinterpret_cast<float*>(wb + ly.off_tbuf) : nullptr;
  __half* xt_hi = DEC ? reinterpret_cast<__half*>(wb + ly.off_xthi) : nullptr;
  __half* xt_lo = DEC ? reinterpret_cast<__half*>(wb + ly.off_xtlo) : nullptr;
  if (lane == 0) mbar_init(xbar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  {
    // zero the fp16 operand tiles once: padding rows (>= N) and columns (>= S) stay 0
    uint32_t* p = reinterpret_cast<uint32_t*>(x_hi);
    const int words = (int)(reinterpret_cast<unsigned char*>(dsc) -
                            reinterpret_cast<unsigned char*>(x_hi)) / 4;
    for (int k = lane; k < words; k += 32) p[k] = 0u;
    if constexpr (DEC) {
      uint32_t* pt = reinterpret_cast<uint32_t*>(xt_hi);
      const int wt_ = (ly.per_warp_bytes - ly.off_xthi) / 4;
      for (int k = lane; k < wt_; k += 32) pt[k] = 0u;
    }
    // S = 24: fp32 staging rows >= N are never loaded and stay 0, so the descriptor phase
    // runs on all lanes without a branch (padding rows give zero X', Z' rows)
    if (SC == 24)
      for (int k = N * S + lane; k < NR * S; k += 32) xbuf[k] = 0.f;
  }
  __syncthreads();

  const bool vec_x = a.x_vec;
  const int NS = N * S;
  // one bulk TMA per series when its segmented span is 16-byte aligned and sized
  const bool bulk = vec_x && ((NS & 3) == 0);
  // S = 24: the output row is staged in the Z' region (free after the Gram) and written
  // by one 1-D TMA bulk store when it is whole float4s (y is 16-byte aligned by contract)
  // (the epilogue writes whole 16-row tiles there: rows >= M land past H and are not stored)
  const bool bstore = SC == 24 && (H & 3) == 0 && 16 * MMT * SC * 4 <= 2 * KO.zhi_bytes;
  uint32_t xphase = 0;
  const int64_t b_begin = (int64_t)blockIdx.x * wins_per_cta;
  int64_t b_end = b_begin + wins_per_cta;
  if (b_end > a.B) b_end = a.B;

  auto prefetch = [&](int64_t b) {
    const float* xg = a.x + b * a.xsb + c * a.xsc + a.r;
    if (bulk) {
      if (lane == 0) bulk_load(xbuf, xg, (uint32_t)NS * 4u, xbar);
      return;
    }
    if (vec_x) {
      for (int k = lane; k < (NS >> 2); k += 32) cp_async16(xbuf + 4 * k, xg + 4 * k);
      for (int k = (NS & ~3) + lane; k < NS; k += 32) cp_async4(xbuf + k, xg + k);
    } else {
      for (int k = lane; k < NS; k += 32) cp_async4(xbuf + k, xg + k);
    }
    cp_async_commit();
  };

  // fold helper: Q' += W'[:, col0 + 16 kt ...] * B  for one k-tile (B = attention tile kt)
  auto fold_tile = [&](float (&qa)[MMT][2 * MT][4], int col0, int kt,
                       const uint32_t (&bh)[2 * MT][2], const uint32_t (&bl)[2 * MT][2]) {
#pragma unroll
    for (int mm = 0; mm < MMT; mm++) {
      uint32_t wh[4], wl[4];
      const int off = (16 * mm + (lane & 7) + 8 * (q8 & 1)) * WPH + col0 + 16 * kt + 8 * (q8 >> 1);
      ldsm_x4(wh, w_hi + off);
      ldsm_x4(wl, w_lo + off);
#pragma unroll
      for (int nt = 0; nt < 2 * MT; nt++) mma16816(qa[mm][nt], wl, bh[nt][0], bh[nt][1]);
#pragma unroll
      for (int nt = 0; nt < 2 * MT; nt++) mma16816(qa[mm][nt], wh, bl[nt][0], bl[nt][1]);
#pragma unroll
      for (int nt = 0; nt < 2 * MT; nt++) mma16816(qa[mm][nt], wh, bh[nt][0], bh[nt][1]);
    }
  };

  int64_t b = b_begin + warp;
  if (b < b_end) prefetch(b);
  for (; b < b_end; b += nwarps) {
    const int64_t series = b * C + c;
    if (bulk) {
      mbar_wait(xbar, xphase);
      xphase ^= 1u;
    } else {
      cp_async_wait_all();
    }
    __syncwarp();

    // ---------------- a2: descriptors (Def 4-5) from d = x - x0 (x0 = the segment's first
    // value, so a constant segment gives exact zeros); X' = x sx, Z' = z sz as fp16 hi/lo
    const int i = lane;
    float x0 = 0.f, m1 = 0.f, mu = 0.f, kap = 0.f, nu2 = 0.f, sx, sz;
    // generic path only: Def 5 pieces computed before pass 2, and the instance-norm map
    // (rr = 1, sr = 1, mr = 0 when off; the S = 24 instantiations never see the widening)
    float gen_mbar = 0.f, gen_var = 0.f, rr = 1.f, sr = 1.f, mr = 0.f;
    // trend-branch level and slope (differ from mu, kap only under DEC)
    float mu_t = 0.f, kap_t = 0.f;
    if constexpr (SC == 24) {
      // lane i holds its whole segment in registers: one read, 16-byte row stores
      float xv[24];
      float2 s1 = f2(0.f), s3 = f2(0.f);
      float amx = 0.f, dmx = 0.f;
      const bool row_ok = MT == 2 || i < NR;   // lanes past NR own no row (MT = 1)
      if (row_ok) {
        const float4* xr = reinterpret_cast<const float4*>(xbuf + i * 24);
#pragma unroll
        for (int q = 0; q < 6; q++) {
          const float4 v = xr[q];
          xv[4 * q] = v.x;
          xv[4 * q + 1] = v.y;
          xv[4 * q + 2] = v.z;
          xv[4 * q + 3] = v.w;
        }
        x0 = xv[0];
#pragma unroll
        for (int t = 0; t < 24; t += 2) {
          const float2 d = add2(make_float2(xv[t], xv[t + 1]), f2(-x0));
          s1 = add2(s1, d);
          s3 = fma2(make_float2((float)t - 11.5f, (float)t - 10.5f), d, s3);
          amx = fmaxf(amx, fmaxf(fabsf(xv[t]), fabsf(xv[t + 1])));
          dmx = fmaxf(dmx, fmaxf(fabsf(d.x), fabsf(d.y)));
        }
        m1 = (s1.x + s1.y) * (1.f / 24.f);
        mu = x0 + m1;
        kap = (s3.x + s3.y) * a.inv_v;
      }
      sx = pow2_scale(warp_max_nonneg(amx));
      sz = pow2_scale(2.f * warp_max_nonneg(dmx));  // |z| <= 2 max|d|
      if (bstore) {  // the previous series' output store has left the Z' region
        if (lane == 0) bulk_wait_read();
        __syncwarp();
      }
      if (row_ok) {
        const float2 sx2 = f2(sx), sz2 = f2(sz), nx0 = f2(-x0), nm1 = f2(-m1);
        float2 q2 = f2(0.f);
#pragma unroll
        for (int q = 0; q < 3; q++) {
          uint4 xh, xl, zh, zl;
          uint32_t* pxh = reinterpret_cast<uint32_t*>(&xh);
          uint32_t* pxl = reinterpret_cast<uint32_t*>(&xl);
          uint32_t* pzh = reinterpret_cast<uint32_t*>(&zh);
          uint32_t* pzl = reinterpret_cast<uint32_t*>(&zl);
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const int t = 8 * q + 2 * u;
            const float2 v = make_float2(xv[t], xv[t + 1]);
            const float2 z = add2(add2(v, nx0), nm1);
            q2 = fma2(z, z, q2);
            split2(mul2(v, sx2), pxh[u], pxl[u]);
            split2(mul2(z, sz2), pzh[u], pzl[u]);
          }
          *reinterpret_cast<uint4*>(x_hi + i * 24 + 8 * q) = xh;
          *reinterpret_cast<uint4*>(x_lo + i * 24 + 8 * q) = xl;
          *reinterpret_cast<uint4*>(z_hi + i * 24 + 8 * q) = zh;
          *reinterpret_cast<uint4*>(z_lo + i * 24 + 8 * q) = zl;
        }
        nu2 = q2.x + q2.y;
      }
      __syncwarp();
    } else if constexpr (DEC) {
      // ---- R-f5: trend = moving average of the N S segmented points with the ends
      // repeated, lane-chunked running sums; seasonal = x - trend.  (RevIN commutes with the
      // average: both components are mapped affinely below.)
      {
        const int hk = (a.ma_k - 1) >> 1;
        const int cnk = (NS + 31) >> 5;
        const int i0 = lane * cnk, i1 = min(i0 + cnk, NS);
        if (i0 < i1) {
          float sacc = 0.f;
          for (int d = -hk; d <= hk; d++) sacc += xbuf[min(max(i0 + d, 0), NS - 1)];
          tbuf[i0] = sacc * a.ma_inv;
          for (int q = i0 + 1; q < i1; q++) {
            sacc += xbuf[min(q + hk, NS - 1)] - xbuf[max(q - 1 - hk, 0)];
            tbuf[q] = sacc * a.ma_inv;
          }
        }
      }
      __syncwarp();
      float s1 = 0.f, s3 = 0.f, s1t = 0.f, s3t = 0.f, amx = 0.f, dmx = 0.f, nu2t = 0.f;
      if (i < N) {
        const float* xr = xbuf + i * S;
        const float* tr = tbuf + i * S;
        x0 = xr[0] - tr[0];
        const float x0t = tr[0];
        // lane-rotated row walks (bank conflicts for S a multiple of 8, as in the plain path)
        const int t_start = ((S & 7) == 0 && S >= 24) ? i % S : 0;
        int t = t_start;
        for (int q = 0; q < S; q++, t = (t + 1 == S) ? 0 : t + 1) {
          const float vt = tr[t], vs = xr[t] - vt;
          const float ds = vs - x0, dt = vt - x0t;
          s1 += ds;
          s3 = fmaf((float)t - a.half_s, ds, s3);
          s1t += dt;
          s3t = fmaf((float)t - a.half_s, dt, s3t);
          amx = fmaxf(amx, fmaxf(fabsf(vs), fabsf(vt)));
          dmx = fmaxf(dmx, fabsf(ds));
        }
        m1 = s1 * a.inv_s;
        mu = x0 + m1;
        kap = s3 * a.inv_v;
        const float m1t = s1t * a.inv_s;
        mu_t = x0t + m1t;
        kap_t = s3t * a.inv_v;
        const float kd = a.detrend ? kap : 0.f;
        t = t_start;
        for (int q = 0; q < S; q++, t = (t + 1 == S) ? 0 : t + 1) {
          const float vt = tr[t], vs = xr[t] - vt;
          const float z = fmaf(-kd, (float)t - a.half_s, (vs - x0) - m1);
          nu2 = fmaf(z, z, nu2);
          const float zt = (vt - x0t) - m1t;
          nu2t = fmaf(zt, zt, nu2t);
        }
      }
      if (a.revin) {   // R-f1 statistics of the segmented points themselves
        float sm = 0.f;
        for (int k = lane; k < NS; k += 32) sm += xbuf[k];
        mr = warp_sum(sm) * a.inv_ns;
        float q = 0.f;
        for (int k = lane; k < NS; k += 32) {
          const float d = xbuf[k] - mr;
          q = fmaf(d, d, q);
        }
        const float vr = warp_sum(q) * a.inv_ns;
        rr = rsqrtf(vr + kEpsRevin);
        sr = (vr + kEpsRevin) * rr;
      }
      // Def 5 on the trend branch's input
      gen_mbar = warp_sum(i < N ? mu_t : 0.f) * a.inv_n;
      gen_var = warp_sum(i < N ? nu2t + (float)S * (mu_t - gen_mbar) * (mu_t - gen_mbar) : 0.f) *
                a.inv_ns;
      sx = pow2_scale((warp_max_nonneg(amx) + fabsf(mr)) * rr);
      sz = 1.f;   // Z' is row-normalised (per-row scale in the descriptor array)
      // per-row shift, mean, slope and Z' scale for the coalesced pass, one float4 per row in
      // the (not yet written) descriptor array.  Row-normalised Gram operand:
      // Z'_i = z_i rr / sqrt(nu2_i rr^2 + eps_s), |Z'_i| <= 1, so the split keeps ~22 bits
      // relative to every row (not to the series' largest row)
      dsc[lane] = make_float4(x0, m1, a.detrend ? kap : 0.f,
                              rsqrtf(nu2 * rr * rr + kEpsSeasonal) * rr);
      __syncwarp();
      const float xsc = rr * sx, xoff = -mr * rr * sx;
      for (int k = lane; k < NS; k += 32) {
        const int r = (int)(((float)k + 0.5f) * a.inv_s);
        const int t = k - r * S;
        const float tv = tbuf[k], vs = xbuf[k] - tv;
        const float4 ri = dsc[r];
        const float xr0 = ri.x, mrow = ri.y, krow = ri.z;
        __half h, l;
        split1(vs * xsc, h, l);
        x_hi[r * sph + t] = h;
        x_lo[r * sph + t] = l;
        split1(fmaf(tv, xsc, xoff), h, l);
        xt_hi[r * sph + t] = h;
        xt_lo[r * sph + t] = l;
        split1(fmaf(-krow, (float)t - a.half_s, (vs - xr0) - mrow) * ri.w, h, l);
        z_hi[r * zph + t] = h;
        z_lo[r * zph + t] = l;
      }
      __syncwarp();
    } else {
      // generic S: pass 1 per lane-row, pass 2 coalesced over elements
      float s1 = 0.f, s3 = 0.f, amx = 0.f, dmx = 0.f;
      if (i < N) {
        const float* xr = xbuf + i * S;
        x0 = xr[0];
        auto acc1 = [&](float v, int t) {
          const float d = v - x0;
          s1 += d;
          s3 = fmaf((float)t - a.half_s, d, s3);
          amx = fmaxf(amx, fabsf(v));
          dmx = fmaxf(dmx, fabsf(d));
        };
        // rows are S floats apart: for S a multiple of 8 the lanes share banks (8-way at
        // S = 24, 32-way at S = 96), so lane i walks its row from column (i mod S) on,
        // wrapping, which spreads the lanes over the banks (A/B: S = 48 1.20 -> 1.00 ms,
        // S = 96 3.30 -> 2.41 ms; at S = 12 the wrap bookkeeping measured slower)
        const bool rot = (S & 7) == 0 && S >= 24;
        if ((S & 3) == 0 && !rot) {
          for (int t = 0; t < S; t += 4) {
            const float4 v = *reinterpret_cast<const float4*>(xr + t);
            acc1(v.x, t);
            acc1(v.y, t + 1);
            acc1(v.z, t + 2);
            acc1(v.w, t + 3);
          }
        } else if ((S & 3) == 0) {
          const int S4 = S >> 2;
          int tq = i % S4;
          for (int q = 0; q < S4; q++) {
            const float4 v = *reinterpret_cast<const float4*>(xr + 4 * tq);
            acc1(v.x, 4 * tq);
            acc1(v.y, 4 * tq + 1);
            acc1(v.z, 4 * tq + 2);
            acc1(v.w, 4 * tq + 3);
            if (++tq == S4) tq = 0;
          }
        } else if (!rot) {
          for (int t = 0; t < S; t++) acc1(xr[t], t);
        } else {
          int t = i % S;
          for (int q = 0; q < S; q++) {
            acc1(xr[t], t);
            if (++t == S) t = 0;
          }
        }
        m1 = s1 * a.inv_s;
        mu = x0 + m1;
        kap = s3 * a.inv_v;
        // nu2: |z|^2, or with metric_variant bit 1 the residual |e|^2, e = z - kappa t~
        // (SURVEY §8(f) f3); Def 5 below uses |z|^2 = |e|^2 + kappa^2 V
        const float kd = a.detrend ? kap : 0.f;
        if (rot) {
          int t = i % S;
          for (int q = 0; q < S; q++) {
            const float z = fmaf(-kd, (float)t - a.half_s, (xr[t] - x0) - m1);
            nu2 = fmaf(z, z, nu2);
            if (++t == S) t = 0;
          }
        } else {
          for (int t = 0; t < S; t++) {
            const float z = fmaf(-kd, (float)t - a.half_s, (xr[t] - x0) - m1);
            nu2 = fmaf(z, z, nu2);
          }
        }
      }
      // sigma^2 (Def 5) and, with instance_norm (f1, R-f1), the RevIN map xhat = (x - mu_r) rr
      gen_mbar = warp_sum(i < N ? mu : 0.f) * a.inv_n;
      {
        const float nz2 = a.detrend ? fmaf(s3, kap, nu2) : nu2;
        gen_var = warp_sum(i < N ? nz2 + (float)S * (mu - gen_mbar) * (mu - gen_mbar) : 0.f) *
                  a.inv_ns;
      }
      if (a.revin) {
        rr = rsqrtf(gen_var + kEpsRevin);
        sr = (gen_var + kEpsRevin) * rr;
        mr = gen_mbar;
      }
      sx = pow2_scale((warp_max_nonneg(amx) + fabsf(mr)) * rr);
      // |e| <= |z| + |kappa| max|t~| <= 2 max|d| + |kappa| (S-1)/2
      sz = 1.f;   // Z' is row-normalised (per-row scale in the descriptor array)
      // per-row shift, mean, slope and row-normalised Z' scale for the coalesced pass (no
      // shuffles in its lane-divergent loop), one float4 per row in the descriptor array
      dsc[lane] = make_float4(x0, m1, a.detrend ? kap : 0.f,
                              rsqrtf(nu2 * rr * rr + kEpsSeasonal) * rr);
      __syncwarp();
      const float xsc = rr * sx, xoff = -mr * rr * sx;
      for (int k = lane; k < NS; k += 32) {
        const int r = (int)(((float)k + 0.5f) * a.inv_s);
        const int t = k - r * S;
        const float v = xbuf[k];
        const float4 ri = dsc[r];
        const float xr0 = ri.x, mrow = ri.y, krow = ri.z;
        __half h, l;
        split1(fmaf(v, xsc, xoff), h, l);
        x_hi[r * sph + t] = h;
        x_lo[r * sph + t] = l;
        split1(fmaf(-krow, (float)t - a.half_s, (v - xr0) - mrow) * ri.w, h, l);
        z_hi[r * zph + t] = h;
        z_lo[r * zph + t] = l;
      }
      __syncwarp();
    }
    if constexpr (!DEC) {
      mu_t = mu;
      kap_t = kap;
    }
    // xbuf is free: fetch the next series while this one is in the tensor cores
    if (b + nwarps < b_end) prefetch(b + nwarps);
    // Def 5: sigma^2 = (1/(N S)) sum_n [nu2_n + S (mu_n - mubar)^2]
    float inv_var;
    if constexpr (SC > 0) {
      const float mbar = warp_sum(i < N ? mu : 0.f) * a.inv_n;
      const float dv = i < N ? nu2 + (float)S * (mu - mbar) * (mu - mbar) : 0.f;
      inv_var = fast_rcp(warp_sum(dv) * a.inv_ns + kEpsTrend);
    } else {
      // of the (normalised) input: var rr^2
      inv_var = fast_rcp(fmaf(gen_var * rr, rr, kEpsTrend));
    }
    {
      // trend: mu~ = mu sqrt(inv_var kt), k~ = kappa sqrt(vtrend inv_var kt) (Def 7-8);
      // seasonal: inv = 1/sqrt(nu2 + eps_s) (Def 6) and the known row maximum f = nu inv:
      // rho_ij <= f_i f_j <= f_i (Cauchy-Schwarz), rho_ii = f_i^2 within f_i (1 - f_i) <= 1/4
      // of it, so exp((rho_ij - f_i) / tau_s) never overflows and its largest term never
      // underflows for tau_s > 0.003; softmax is shift-invariant, so this is the same result
      // as subtracting the searched max (Def 8).
      // (MUFU square roots: a common relative factor per series, <= ~1 ulp)
      const float cmr = fast_sqrt(inv_var * a.kt);
      const float cm = cmr * rr, ck = cmr * fast_sqrt(a.vtrend) * rr;
      // seasonal normaliser of the normalised input: 1/sqrt(nu2 rr^2 + eps_s); the Gram is of
      // z sz (unnormalised), so the column factor carries one rr and rk the other
      const float nh2 = nu2 * rr * rr;
      const float invh = rsqrtf(nh2 + kEpsSeasonal);
      // generic path: the Gram of the row-normalised Z' is rho itself (column factor 1)
      dsc[lane] = i < N ? make_float4((mu_t - mr) * cm, kap_t * ck, SC == 0 ? 1.f : invh * rr,
                                      fast_sqrt(nh2) * invh)
                        : make_float4(0.f, 0.f, 1.f, 0.f);
      if ((SC == 0 || COMP) && a.comp) {   // the (normalised) segment levels and slopes
        cvec[lane] = i < N ? (DEC ? mu : mu - mr) * rr : 0.f;
        cvec[32 + lane] = i < N ? kap * rr : 0.f;
        cvec[256 + lane] = i < N ? (mu_t - mr) * rr : 0.f;
        cvec[288 + lane] = i < N ? kap_t * rr : 0.f;
      }
      __syncwarp();
    }

    // component values (generic path): row ii of A times mu^ and kappa^, reduced over the
    // quad's 4 lanes, into cvec[dst + ii], cvec[dst + 32 + ii]
    const bool comp = (SC == 0 || COMP) && a.comp != 0;
    auto comp_rows = [&](const float2 (&p)[2 * MT], int ii, int dst, int src) {
      float2 am = f2(0.f), ak = f2(0.f);
#pragma unroll
      for (int nt = 0; nt < 2 * MT; nt++) {
        const int j = 8 * nt + 2 * cq;
        am = fma2(p[nt], make_float2(cvec[src + j], cvec[src + j + 1]), am);
        ak = fma2(p[nt], make_float2(cvec[src + 32 + j], cvec[src + 33 + j]), ak);
      }
      float sm = am.x + am.y, sk = ak.x + ak.y;
      sm += __shfl_xor_sync(0xffffffffu, sm, 1);
      sk += __shfl_xor_sync(0xffffffffu, sk, 1);
      sm += __shfl_xor_sync(0xffffffffu, sm, 2);
      sk += __shfl_xor_sync(0xffffffffu, sk, 2);
      if (cq == 0) {
        cvec[dst + ii] = ii < N ? sm : 0.f;
        cvec[dst + 32 + ii] = ii < N ? sk : 0.f;
      }
    };

    float qa[MMT][2 * MT][4];  // Q' = sw (W_s A_s + W_t A_t)   (component values: sw W_s A_s)
    float qa2[DEC ? MMT : 1][2 * MT][4];   // DEC: Q_t' = sw W_t A_t (its own head operand)
#pragma unroll
    for (int mm = 0; mm < MMT; mm++)
#pragma unroll
      for (int nt = 0; nt < 2 * MT; nt++)
#pragma unroll
        for (int e = 0; e < 4; e++) qa[mm][nt][e] = 0.f;
    if constexpr (DEC) {
#pragma unroll
      for (int mm = 0; mm < MMT; mm++)
#pragma unroll
        for (int nt = 0; nt < 2 * MT; nt++)
#pragma unroll
          for (int e = 0; e < 4; e++) qa2[mm][nt][e] = 0.f;
    }

    // ---------------- a4+a5 trend: exponent -Dhat_ij / tau_t (row max is 0 at j = i,
    // D_ii = 0) = -(mu~_i - mu~_j)^2 - (k~_i - k~_j)^2 with mu~ = mu sqrt(inv_var kt),
    // k~ = kappa sqrt(vtrend inv_var kt) (Def 7-8); then fold Q' += W'_t A_t per k-tile
    {
      float2 cmu[2 * MT], ckap[2 * MT];
#pragma unroll
      for (int nt = 0; nt < 2 * MT; nt++) {
        const int j = 8 * nt + 2 * cq;
        const float4 d0 = dsc[j], d1 = dsc[j + 1];
        cmu[nt] = make_float2(j < N ? -d0.x : -INFINITY, j + 1 < N ? -d1.x : -INFINITY);
        ckap[nt] = make_float2(-d0.y, -d1.y);
      }
#pragma unroll
      for (int mt = 0; mt < MT; mt++) {
        uint32_t bh[2 * MT][2], bl[2 * MT][2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int ii = 16 * mt + 8 * h + gq;
          const float4 di = dsc[ii];
          const float2 mui = f2(di.x), ki = f2(di.y);
          float2 u[2 * MT];
          float2 sum2 = f2(0.f);
#pragma unroll
          for (int nt = 0; nt < 2 * MT; nt++) {
            const float2 dm = add2(mui, cmu[nt]), dk = add2(ki, ckap[nt]);
            const float2 e = fma2(make_float2(-dk.x, -dk.y), dk, mul2(make_float2(-dm.x, -dm.y), dm));
            u[nt] = make_float2(fast_ex2(e.x), fast_ex2(e.y));
            sum2 = add2(sum2, u[nt]);
          }
          float sum = sum2.x + sum2.y;
          sum += __shfl_xor_sync(0xffffffffu, sum, 1);
          sum += __shfl_xor_sync(0xffffffffu, sum, 2);
          const float2 rs2 = f2(ii < N ? fast_rcp(sum) : 0.f);
          if (comp) {
            float2 pr[2 * MT];
#pragma unroll
            for (int nt = 0; nt < 2 * MT; nt++) pr[nt] = mul2(u[nt], rs2);
            comp_rows(pr, ii, 128, 256);
          }
#pragma unroll
          for (int nt = 0; nt < 2 * MT; nt++) {
            const float2 p = mul2(u[nt], rs2);
            if constexpr (DBG) {
              if (ii < N) {
                const int j = 8 * nt + 2 * cq;
                float* d = a.a_t_dbg + (series * N + ii) * N + j;
                if (j < N) d[0] = p.x;
                if (j + 1 < N) d[1] = p.y;
              }
            }
            uint32_t hi, lo;
            split2(p, hi, lo);
            bh[nt][h] = movm_t(hi);
            bl[nt][h] = movm_t(lo);
          }
        }
        if (!comp) {
          if constexpr (DEC) fold_tile(qa2, NR, mt, bh, bl);
          else fold_tile(qa, NR, mt, bh, bl);
        }
      }
    }

    // ---------------- a3 + a5 seasonal, one 16-row tile of query segments at a time:
    // Gram rows G'[16 mt .. 16 mt + 15][:] = Z' Z'^T (= sz^2 G), rho_ij = G'_ij inv_i inv_j / sz^2
    // with inv = 1/sqrt(nu2 + eps_s) (Def 6), row softmax on the fragments, fold Q' += W'_s A_s
    {
      const float ks_z = SC == 0 ? a.ks : a.ks * fast_rcp(sz * sz);   // sz^2: a power of two
      float2 cinv[2 * MT], cmask[2 * MT];
#pragma unroll
      for (int nt = 0; nt < 2 * MT; nt++) {
        const int j = 8 * nt + 2 * cq;
        cinv[nt] = make_float2(dsc[j].z, dsc[j + 1].z);
        cmask[nt] = make_float2(j < N ? 0.f : -INFINITY, j + 1 < N ? 0.f : -INFINITY);
      }
      const int k16 = SC > 0 ? (SC / 16) * 16 : ly.kz;
#pragma unroll
      for (int mt = 0; mt < MT; mt++) {
        float g[2 * MT][4];
#pragma unroll
        for (int nt = 0; nt < 2 * MT; nt++)
#pragma unroll
          for (int e = 0; e < 4; e++) g[nt][e] = 0.f;
        for (int k0 = 0; k0 < k16; k0 += 16) {
          uint32_t ah[4], al[4];
          {
            const int off = (16 * mt + (lane & 7) + 8 * (q8 & 1)) * zph + k0 + 8 * (q8 >> 1);
            ldsm_x4(ah, z_hi + off);
            ldsm_x4(al, z_lo + off);
          }
#pragma unroll
          for (int np = 0; np < MT; np++) {
            uint32_t bh[4], bl[4];
            const int off = (16 * np + (lane & 7) + 8 * (q8 >> 1)) * zph + k0 + 8 * (q8 & 1);
            ldsm_x4(bh, z_hi + off);
            ldsm_x4(bl, z_lo + off);
            // product-major order: independent accumulators back to back
            mma16816(g[2 * np], al, bh[0], bh[1]);
            mma16816(g[2 * np + 1], al, bh[2], bh[3]);
            mma16816(g[2 * np], ah, bl[0], bl[1]);
            mma16816(g[2 * np + 1], ah, bl[2], bl[3]);
            mma16816(g[2 * np], ah, bh[0], bh[1]);
            mma16816(g[2 * np + 1], ah, bh[2], bh[3]);
          }
        }
        if constexpr (SC > 0 && (SC % 16) == 8) {
          // K tail of 8 (S = 24: columns 16..23) with m16n8k8
          constexpr int kt0 = (SC / 16) * 16;
          uint32_t ah[2], al[2];
          {
            const int off = (16 * mt + (lane & 7) + 8 * (q8 & 1)) * zph + kt0;
            ldsm_x2(ah[0], ah[1], z_hi + off);
            ldsm_x2(al[0], al[1], z_lo + off);
          }
#pragma unroll
          for (int np = 0; np < MT; np++) {
            uint32_t bh[2], bl[2];  // b0 of n-tiles 2np, 2np+1 (rows j of Z', k = 16..23)
            const int off = (16 * np + 8 * (q8 & 1) + (lane & 7)) * zph + kt0;
            ldsm_x2(bh[0], bh[1], z_hi + off);
            ldsm_x2(bl[0], bl[1], z_lo + off);
            mma1688(g[2 * np], al[0], al[1], bh[0]);
            mma1688(g[2 * np + 1], al[0], al[1], bh[1]);
            mma1688(g[2 * np], ah[0], ah[1], bl[0]);
            mma1688(g[2 * np + 1], ah[0], ah[1], bl[1]);
            mma1688(g[2 * np], ah[0], ah[1], bh[0]);
            mma1688(g[2 * np + 1], ah[0], ah[1], bh[1]);
          }
        }
        uint32_t bh[2 * MT][2], bl[2 * MT][2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int ii = 16 * mt + 8 * h + gq;
          const float4 di = dsc[ii];
          const float rk = di.z * ks_z;
          float2 u[2 * MT];
#pragma unroll
          for (int nt = 0; nt < 2 * MT; nt++)
            u[nt] = fma2(make_float2(g[nt][2 * h], g[nt][2 * h + 1]), cinv[nt], cmask[nt]);
          const float2 rk2 = f2(rk), nb2 = f2(-di.w * a.ks);
          float2 sum2 = f2(0.f);
#pragma unroll
          for (int nt = 0; nt < 2 * MT; nt++) {
            const float2 arg = fma2(u[nt], rk2, nb2);
            u[nt] = make_float2(fast_ex2(arg.x), fast_ex2(arg.y));
            sum2 = add2(sum2, u[nt]);
          }
          float sum = sum2.x + sum2.y;
          sum += __shfl_xor_sync(0xffffffffu, sum, 1);
          sum += __shfl_xor_sync(0xffffffffu, sum, 2);
          const float2 rs2 = f2(ii < N ? fast_rcp(sum) : 0.f);
          if (comp) {
            float2 pr[2 * MT];
#pragma unroll
            for (int nt = 0; nt < 2 * MT; nt++) pr[nt] = mul2(u[nt], rs2);
            comp_rows(pr, ii, 64, 0);
          }
#pragma unroll
          for (int nt = 0; nt < 2 * MT; nt++) {
            const float2 p = mul2(u[nt], rs2);
            if constexpr (DBG) {
              if (ii < N) {
                const int j = 8 * nt + 2 * cq;
                float* d = a.a_s_dbg + (series * N + ii) * N + j;
                if (j < N) d[0] = p.x;
                if (j + 1 < N) d[1] = p.y;
              }
            }
            uint32_t hi, lo;
            split2(p, hi, lo);
            bh[nt][h] = movm_t(hi);
            bl[nt][h] = movm_t(lo);
          }
        }
        fold_tile(qa, 0, mt, bh, bl);
      }
    }

    // ---------------- a7 head Y' = Q' X' (= sw sx Y), one 16-row tile of future segments
    // at a time, t in chunks of 4 tiles; a8 store y = Y + b
    // the output staging row (bstore) overwrites the Z' tiles the Gram's ldmatrix just read
    // (other lanes' rows): order the two explicitly
    if (bstore) __syncwarp();
    if (comp) {
      // Y = W_s A_s V_s + W_t A_t V_t with V_s = X^ - mu^ - d1 kappa^ t~, V_t = mu^ + d0 kappa^ t~
      //   = (W_s A_s) X^ + alpha_m + beta_m t~      (d1 = bit 1, d0 = 1 - bit 0)
      // alpha = W_t (A_t mu^) - W_s (A_s mu^), beta = d0 W_t (A_t kappa^) - d1 W_s (A_s kappa^);
      // W from the packed head (W' = W sw as fp16 hi + lo), stored times sr (de-normalised)
      __syncwarp();
      const int m = lane;
      float al = 0.f, be = 0.f;
      if (m < M) {
        const float d0 = a.vtrend != 0.f ? 1.f : 0.f, d1 = a.detrend ? 1.f : 0.f;
        for (int n = 0; n < N; n++) {
          const float ws_ = __half2float(w_hi[m * WPH + n]) + __half2float(w_lo[m * WPH + n]);
          const float wt_ =
              __half2float(w_hi[m * WPH + NR + n]) + __half2float(w_lo[m * WPH + NR + n]);
          al = fmaf(wt_, cvec[128 + n], fmaf(-ws_, cvec[64 + n], al));
          be = fmaf(d0 * wt_, cvec[160 + n], fmaf(-d1 * ws_, cvec[96 + n], be));
        }
      }
      cvec[192 + lane] = al * inv_sw * sr;
      cvec[224 + lane] = be * inv_sw * sr;
      __syncwarp();
    }
    const float2 ys2 = f2(inv_sw * sr / sx);
    const bool pair_store = ((S | H) & 1) == 0;   // t, hh even -> 8-byte aligned pairs
    float* yg = a.y + series * H;
    float* ystage = reinterpret_cast<float*>(z_hi);
#pragma unroll
    for (int mm = 0; mm < MMT; mm++) {
      if (16 * mm >= M) break;
      uint32_t qh[MT][4], ql[MT][4];   // Q' fragments -> A operand (hi/lo, in registers)
#pragma unroll
      for (int kj = 0; kj < MT; kj++) {
        split2(qa[mm][2 * kj][0], qa[mm][2 * kj][1], qh[kj][0], ql[kj][0]);
        split2(qa[mm][2 * kj][2], qa[mm][2 * kj][3], qh[kj][1], ql[kj][1]);
        split2(qa[mm][2 * kj + 1][0], qa[mm][2 * kj + 1][1], qh[kj][2], ql[kj][2]);
        split2(qa[mm][2 * kj + 1][2], qa[mm][2 * kj + 1][3], qh[kj][3], ql[kj][3]);
      }
      uint32_t qh2[DEC ? MT : 1][4], ql2[DEC ? MT : 1][4];   // DEC: Q_t' fragments
      if constexpr (DEC) {
#pragma unroll
        for (int kj = 0; kj < MT; kj++) {
          split2(qa2[mm][2 * kj][0], qa2[mm][2 * kj][1], qh2[kj][0], ql2[kj][0]);
          split2(qa2[mm][2 * kj][2], qa2[mm][2 * kj][3], qh2[kj][1], ql2[kj][1]);
          split2(qa2[mm][2 * kj + 1][0], qa2[mm][2 * kj + 1][1], qh2[kj][2], ql2[kj][2]);
          split2(qa2[mm][2 * kj + 1][2], qa2[mm][2 * kj + 1][3], qh2[kj][3], ql2[kj][3]);
        }
      }
      for (int t0 = 0; t0 < ntt; t0 += 4) {
        float ya[4][4];
#pragma unroll
        for (int nt = 0; nt < 4; nt++)
#pragma unroll
          for (int e = 0; e < 4; e++) ya[nt][e] = 0.f;
#pragma unroll
        for (int kj = 0; kj < MT; kj++) {
#pragma unroll
          for (int tp = 0; tp < 2; tp++) {
            const int nt0 = t0 + 2 * tp;
            if (nt0 >= ntt) break;
            uint32_t xh[4], xl[4];
            const int krow = 16 * kj + (lane & 7) + 8 * (q8 & 1);
            const bool two = nt0 + 1 < ntt;
            if (two) {
              const int off = krow * sph + 8 * (nt0 + (q8 >> 1));
              ldsm_x4_t(xh, x_hi + off);
              ldsm_x4_t(xl, x_lo + off);
            } else {
              const int off = krow * sph + 8 * nt0;
              ldsm_x2_t(xh[0], xh[1], x_hi + off);
              ldsm_x2_t(xl[0], xl[1], x_lo + off);
              xh[2] = xh[3] = xl[2] = xl[3] = 0u;
            }
            mma16816(ya[2 * tp], ql[kj], xh[0], xh[1]);
            if (two) mma16816(ya[2 * tp + 1], ql[kj], xh[2], xh[3]);
            mma16816(ya[2 * tp], qh[kj], xl[0], xl[1]);
            if (two) mma16816(ya[2 * tp + 1], qh[kj], xl[2], xl[3]);
            mma16816(ya[2 * tp], qh[kj], xh[0], xh[1]);
            if (two) mma16816(ya[2 * tp + 1], qh[kj], xh[2], xh[3]);
            if constexpr (DEC) {
              if (!comp) {   // + Q_t' X_t'
                if (two) {
                  const int off = krow * sph + 8 * (nt0 + (q8 >> 1));
                  ldsm_x4_t(xh, xt_hi + off);
                  ldsm_x4_t(xl, xt_lo + off);
                } else {
                  const int off = krow * sph + 8 * nt0;
                  ldsm_x2_t(xh[0], xh[1], xt_hi + off);
                  ldsm_x2_t(xl[0], xl[1], xt_lo + off);
                }
                mma16816(ya[2 * tp], ql2[kj], xh[0], xh[1]);
                if (two) mma16816(ya[2 * tp + 1], ql2[kj], xh[2], xh[3]);
                mma16816(ya[2 * tp], qh2[kj], xl[0], xl[1]);
                if (two) mma16816(ya[2 * tp + 1], qh2[kj], xl[2], xl[3]);
                mma16816(ya[2 * tp], qh2[kj], xh[0], xh[1]);
                if (two) mma16816(ya[2 * tp + 1], qh2[kj], xh[2], xh[3]);
              }
            }
          }
        }
        if (bstore) {
          // whole tiles into the staging row (bias zero-padded): no masks, no branches
#pragma unroll
          for (int nt = 0; nt < (SC + 7) / 8; nt++) {
            if (nt >= 4) break;
#pragma unroll
            for (int h = 0; h < 2; h++) {
              const int hh = (16 * mm + 8 * h + gq) * SC + 8 * (t0 + nt) + 2 * cq;
              const float2 v = mul2(make_float2(ya[nt][2 * h], ya[nt][2 * h + 1]), ys2);
              float2 bb = *reinterpret_cast<const float2*>(bS + hh);
              if (comp) {   // + alpha_m + beta_m t~ (component values)
                const int m = 16 * mm + 8 * h + gq;
                const float t = (float)(8 * (t0 + nt) + 2 * cq) - a.half_s;
                bb = add2(bb, fma2(f2(cvec[224 + m]), make_float2(t, t + 1.f), f2(cvec[192 + m])));
              }
              *reinterpret_cast<float2*>(ystage + hh) = add2(v, bb);
            }
          }
          continue;
        }
#pragma unroll
        for (int nt = 0; nt < 4; nt++) {
          const int t = 8 * (t0 + nt) + 2 * cq;
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int m = 16 * mm + 8 * h + gq;
            if (m < M && t < S) {
              const int hh = m * S + t;
              const float2 v = mul2(make_float2(ya[nt][2 * h], ya[nt][2 * h + 1]), ys2);
              if (pair_store) {  // hh even, H even: hh < H implies hh + 1 < H
                if (hh >= H) continue;
                float2 bb = *reinterpret_cast<const float2*>(bS + hh);
                if (SC == 0 && a.revin) bb = fma2(bb, f2(sr), f2(mr));   // y = yhat sr + mr
                if (comp)
                  bb = add2(bb, fma2(f2(cvec[224 + m]),
                                     make_float2((float)t - a.half_s, (float)t + 1.f - a.half_s),
                                     f2(cvec[192 + m])));
                const float2 o = add2(v, bb);
                asm volatile("st.global.cs.v2.f32 [%0], {%1,%2};" ::"l"(yg + hh), "f"(o.x),
                             "f"(o.y)
                             : "memory");
              } else {
                float c0 = 0.f, c1 = 0.f;
                if (comp) {
                  c0 = fmaf(cvec[224 + m], (float)t - a.half_s, cvec[192 + m]);
                  c1 = fmaf(cvec[224 + m], (float)t + 1.f - a.half_s, cvec[192 + m]);
                }
                if (hh < H) yg[hh] = v.x + fmaf(bS[hh], sr, mr) + c0;
                if (t + 1 < S && hh + 1 < H) yg[hh + 1] = v.y + fmaf(bS[hh + 1], sr, mr) + c1;
              }
            }
          }
        }
      }
    }
    if (bstore) {
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) bulk_store(yg, ystage, (uint32_t)H * 4u);
    }
  }
  cp_async_wait_all();
  if (bstore && lane == 0) bulk_wait_all();
}

int mma_wpack_bytes(int N, int M) {
  const int nr = N <= 16 ? 16 : 32, rows = M <= 16 ? 16 : 32, wph = 2 * nr + 8;
  return ((2 * rows * wph * 2) + 15) & ~15;
}

void pack_mma_head(const float* ws, const float* wt, int Cw, int M, int N, unsigned char* out,
                   float* inv_sw) {
  const int nr = N <= 16 ? 16 : 32, rows = M <= 16 ? 16 : 32, wph = 2 * nr + 8;
  const int bytes = mma_wpack_bytes(N, M);
  for (int c = 0; c < Cw; c++) {
    const float* s = ws + (size_t)c * M * N;
    const float* t = wt + (size_t)c * M * N;
    float mx = 0.f;
    for (int k = 0; k < M * N; k++) mx = fmaxf(mx, fmaxf(fabsf(s[k]), fabsf(t[k])));
    float sw = 1.f;
    if (mx > 0.f && std::isfinite(mx)) {
      int e;
      frexpf(mx, &e);
      sw = ldexpf(1.f, -e);
    }
    inv_sw[c] = 1.f / sw;
    __half* hi = reinterpret_cast<__half*>(out + (size_t)c * bytes);
    __half* lo = hi + rows * wph;
    for (int m = 0; m < rows; m++)
      for (int col = 0; col < wph; col++) {
        float v = 0.f;
        if (m < M) {
          if (col < nr) {
            if (col < N) v = s[m * N + col] * sw;
          } else if (col < 2 * nr) {
            if (col - nr < N) v = t[m * N + (col - nr)] * sw;
          }
        }
        const __half h = __float2half_rn(v);
        hi[m * wph + col] = h;
        lo[m * wph + col] = __float2half_rn(v - __half2float(h));
      }
  }
}

static int odd8(int halves) {  // round up to a multiple of 8 halves whose /8 is odd
  int v = (halves + 7) & ~7;
  if (((v / 8) & 1) == 0) v += 8;
  return v;
}

bool plan_mma_kernel(const FwdArgs& a, int max_smem_optin, MmaPlan* p) {
  if (a.N < 1 || a.N > 32 || a.M > 32 || a.S > 128) return false;
  MmaLayout& ly = p->ly;
  p->mt = a.N <= 16 ? 1 : 2;
  p->mmt = a.M <= 16 ? 1 : 2;
  // the S = 24 instantiations implement the plain reading only (the widening runs generic)
  p->sc = (a.S == 24 && !a.detrend && !a.revin && a.ma_k == 0) ? 24 : 0;
  p->dec = a.ma_k > 0;
  ly.nr = 16 * p->mt;
  if (p->sc == 24) {  // dense rows of 24 halves (48 B: 16-byte aligned, conflict-free ldmatrix)
    ly.sph = 24;
    ly.kz = 24;
    ly.zph = 24;
  } else {
    ly.sph = odd8(a.S);
    ly.kz = (a.S + 15) & ~15;
    ly.zph = odd8(ly.kz);
  }
  ly.wph = 2 * ly.nr + 8;
  ly.ntt = (a.S + 7) / 8;
  const MmaOffsets o =
      mma_offsets(ly.nr, a.S, ly.sph, ly.zph, p->mmt, (p->sc == 0 || a.comp) ? kCompBytes : 0);
  ly.xbuf_f = ly.nr * a.S;
  ly.off_xhi = o.xhi;
  ly.off_xlo = o.xlo;
  ly.off_zhi = o.zhi;
  ly.off_zlo = o.zlo;
  ly.off_diag = o.misc;
  ly.per_warp_bytes = o.pw;
  ly.off_wlo = o.wlo;
  ly.wpack_bytes = o.wpack;
  ly.off_bias = -1;  // after the per-warp regions (depends on warps per CTA)
  ly.off_tbuf = ly.off_xthi = ly.off_xtlo = -1;
  if (p->dec) {   // trend staging and X_t' tiles after the misc region
    ly.off_tbuf = ly.per_warp_bytes;
    ly.off_xthi = r16(ly.off_tbuf + ly.nr * a.S * 4);
    ly.off_xtlo = r16(ly.off_xthi + ly.nr * ly.sph * 2);
    ly.per_warp_bytes = (r16(ly.off_xtlo + ly.nr * ly.sph * 2) + 127) & ~127;
  }
  ly.shared_bytes = o.wpack;
  p->warps_per_cta = PRNET_MMA_THREADS / 32;
  const int hb = a.H > 16 * p->mmt * a.S ? a.H : 16 * p->mmt * a.S;  // zero-padded bias
  auto total = [&](int w) {
    return (size_t)o.wpack + (size_t)w * ly.per_warp_bytes + (size_t)hb * 4;
  };
  while (total(p->warps_per_cta) > (size_t)max_smem_optin && p->warps_per_cta > 1)
    p->warps_per_cta >>= 1;
  p->smem_bytes = total(p->warps_per_cta);
  if (p->smem_bytes > (size_t)max_smem_optin) return false;
  if (p->sc == 24 && mma_wpack_bytes(a.N, a.M) != o.wpack) return false;
  p->wins_per_cta = p->warps_per_cta * 16;
  return true;
}

template <int MT, int MMT, int SC, bool DBG, int NC = 0, bool DEC = false, bool COMP = false>
static cudaError_t launch_t(const FwdArgs& a, const MmaPlan& p, cudaStream_t st) {
  auto k = prnet_fwd_mma_kernel<MT, MMT, SC, DBG, NC, DEC, COMP>;
  cudaError_t e =
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((a.B + p.wins_per_cta - 1) / p.wins_per_cta), (unsigned)a.C);
  k<<<grid, 32 * p.warps_per_cta, p.smem_bytes, st>>>(a, p.ly, p.wins_per_cta);
  return cudaGetLastError();
}

template <int SC, bool DBG, bool DEC = false, bool COMP = false>
static cudaError_t launch_sc(const FwdArgs& a, const MmaPlan& p, cudaStream_t st) {
  if (p.mt == 1)
    return p.mmt == 1 ? launch_t<1, 1, SC, DBG, 0, DEC, COMP>(a, p, st)
                      : launch_t<1, 2, SC, DBG, 0, DEC, COMP>(a, p, st);
  return p.mmt == 1 ? launch_t<2, 1, SC, DBG, 0, DEC, COMP>(a, p, st)
                    : launch_t<2, 2, SC, DBG, 0, DEC, COMP>(a, p, st);
}

cudaError_t launch_mma_kernel(const FwdArgs& a, const MmaPlan& p, cudaStream_t st) {
  const bool dbg = a.a_s_dbg != nullptr;
  if (p.sc == 24 && a.comp && !dbg)   // component values at S = 24 (the attention dump
    // does not depend on them: it runs the plain debug instantiation)
    return launch_sc<24, false, false, true>(a, p, st);
  if (p.sc == 24 && a.N == 30 && !dbg)   // L = 720, S = 24: configs[1..3], plain reading
    return p.mmt == 1 ? launch_t<2, 1, 24, false, 30>(a, p, st)
                      : launch_t<2, 2, 24, false, 30>(a, p, st);
  if (p.sc == 24) return dbg ? launch_sc<24, true>(a, p, st) : launch_sc<24, false>(a, p, st);
  if (p.dec) return dbg ? launch_sc<0, true, true>(a, p, st) : launch_sc<0, false, true>(a, p, st);
  return dbg ? launch_sc<0, true>(a, p, st) : launch_sc<0, false>(a, p, st);
}

}  // namespace prnet
