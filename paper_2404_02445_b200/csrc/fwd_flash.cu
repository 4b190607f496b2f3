// fwd_flash.cu -- PRNet pattern-attention forward for long lookbacks (32 < N <= 512
// segments; the stress sweep of BASELINE.json configs[4], L up to 5760) on the
// tensor cores, flash-attention style.
//
// Same reading and split-fp16 3-product arithmetic as
// fwd_mma.cu.  The N x N similarity matrices are never materialised: one CTA owns
// one series, warps take 16-row query tiles, and for each 16-key tile
//   a3  Gram tile      G' = Z'_i Z'_j^T                      (mma.sync m16n8k16)
//   a4  trend logits   -(mu~_i - mu~_j)^2 - (k~_i - k~_j)^2  (FP32, packed f32x2)
//   a5  exponentials with a KNOWN row maximum -- 0 for the trend row (D_ii = 0) and
//       f_i = nu_i / sqrt(nu2_i + eps_s) >= rho_ij for the seasonal row (Cauchy-Schwarz)
//       -- so no online rescaling is needed; the row sums accumulate
//   a6  P_s += E_s X_j,  P_t += E_t X_j   (E straight from the accumulator fragments
//       to the A operand, FA2 style; X_j from shared memory)      (mma.sync)
// then the 16 pattern rows are normalised and folded into the head accumulator
//   a7  Y += W'_s[:, tile] P_s + W'_t[:, tile] P_t     (P transposed with movmatrix)
// and a fixed-order reduction over the warps adds the bias (a8).
#include <cuda_fp16.h>

#include <cmath>

#include "mma_common.cuh"

// CTAs per SM by register budget: S <= 32 (KS <= 2) and S in (32, 48] (KS = 3) two CTAs at 128
// registers (measured, round 2: KS = 3 spills 200-400 bytes and is still 16-20 % faster, stress
// L2880/S48 3.49 -> 2.91 ms, L2880/S48/H720 4.08 -> 3.25, L5760/S48 9.09 -> 7.61); S > 48 (two
// t-chunks) one CTA (at 128 registers it spills more and was 19-24 % slower, L5760/S96 8.14 ->
// 10.07)
#ifndef PRNET_FLASH_MINB3
#define PRNET_FLASH_MINB3 2
#endif
#ifndef PRNET_FLASH_MINB4
#define PRNET_FLASH_MINB4 1
#endif

namespace prnet {

namespace {

// a hi/lo fp16 pair of consecutive columns (t, t + 1) of a row: one packed split, 4-byte stores;
// the last column of an odd-length row alone
__device__ __forceinline__ void store_split_pair(__half* hi, __half* lo, int o, float v0, float v1,
                                                 bool two) {
  uint32_t h2, l2;
  split2(make_float2(v0, v1), h2, l2);
  if (two) {
    *reinterpret_cast<uint32_t*>(hi + o) = h2;
    *reinterpret_cast<uint32_t*>(lo + o) = l2;
  } else {
    hi[o] = __ushort_as_half((unsigned short)(h2 & 0xFFFFu));
    lo[o] = __ushort_as_half((unsigned short)(l2 & 0xFFFFu));
  }
}

// two block reductions for the price of one pair of barriers (scratch holds 2 nw floats)
__device__ __forceinline__ void block_reduce2(float& u, float& v, float* scratch, bool is_max) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  u = is_max ? warp_max(u) : warp_sum(u);
  v = is_max ? warp_max(v) : warp_sum(v);
  __syncthreads();
  if (lane == 0) {
    scratch[2 * warp] = u;
    scratch[2 * warp + 1] = v;
  }
  __syncthreads();
  float ru = 0.f, rv = 0.f;
  for (int w = 0; w < nw; w++) {
    ru = is_max ? fmaxf(ru, scratch[2 * w]) : ru + scratch[2 * w];
    rv = is_max ? fmaxf(rv, scratch[2 * w + 1]) : rv + scratch[2 * w + 1];
  }
  u = ru;
  v = rv;
}

// A-fragment (16 x 16, rows r0.., cols c0..) of a row-major global fp16 matrix
__device__ __forceinline__ void ldg_afrag(const __half* base, int ld, int r0, int c0, int lane,
                                          uint32_t (&f)[4]) {
  const int g = lane >> 2, c = lane & 3;
  const __half* p = base + (size_t)(r0 + g) * ld + c0 + 2 * c;
  f[0] = __ldg(reinterpret_cast<const unsigned int*>(p));
  f[1] = __ldg(reinterpret_cast<const unsigned int*>(p + 8 * ld));
  f[2] = __ldg(reinterpret_cast<const unsigned int*>(p + 8));
  f[3] = __ldg(reinterpret_cast<const unsigned int*>(p + 8 * ld + 8));
}

}  // namespace

static int flash_npad(int N) { return (N + 15) & ~15; }

// m-rows of the pack: 16 / 32 (the flash kernel, M <= 32), 64 (tc_long only, M <= 64)
static int flash_rows(int M) { return M <= 16 ? 16 : (M <= 32 ? 32 : 64); }
int flash_wpack_bytes(int N, int M) {
  const int rows = flash_rows(M);
  return 2 * rows * 2 * flash_npad(N) * 2;   // hi + lo, [rows][2 Npad] halves
}

// W' = W sw as fp16 hi/lo, row-major [16 MMT][2 Npad]: seasonal i at [0, Npad),
// trend i at [Npad, 2 Npad); hi block then lo block.
void pack_flash_head(const float* ws, const float* wt, int Cw, int M, int N, unsigned char* out,
                     float* inv_sw) {
  const int rows = flash_rows(M), np = flash_npad(N), ld = 2 * np;
  const int bytes = flash_wpack_bytes(N, M);
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
    __half* lo = hi + rows * ld;
    for (int m = 0; m < rows; m++)
      for (int k = 0; k < ld; k++) {
        float v = 0.f;
        if (m < M) {
          if (k < np) {
            if (k < N) v = s[m * N + k] * sw;
          } else if (k - np < N) {
            v = t[m * N + (k - np)] * sw;
          }
        }
        const __half h = __float2half_rn(v);
        hi[m * ld + k] = h;
        lo[m * ld + k] = __float2half_rn(v - __half2float(h));
      }
  }
}

// S <= 32 (KS <= 2): registers capped at 128 so two 8-warp (or four 4-warp) CTAs fit an SM
// (A/B, stress L = 1440, S = 24: 1.84 vs 2.91 ms); S in (32, 48] would spill, keeps 1
// NTT = t tiles of 8 per chunk: S <= 48 in one chunk; longer segments (S <= 96) in
// ly.nch chunks of NTT tiles, the Gram and exponentials recomputed per chunk (the P, Y
// accumulators of all of S would not fit the register file)
// COMP: component values (metric_variant bit 2, reading R-f4): P_s = A_s X - (A_s mu) 1^T -
// d1 (A_s kappa) t~^T and P_t = (A_t mu) 1^T + d0 (A_t kappa) t~^T, from four row sums
// accumulated with the exponentials (no A_t X product)
template <int KS, int NTT, int MMT, bool COMP = false>
__global__ void __launch_bounds__(256, (KS <= 2 ? 2 : (KS == 3 ? PRNET_FLASH_MINB3 : PRNET_FLASH_MINB4))) prnet_fwd_flash_kernel(FwdArgs a, FlashLayout ly,
                                                                 int wins_per_cta) {
  extern __shared__ float4 smem4[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(smem4);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int gq = lane >> 2, cq = lane & 3, q8 = lane >> 3;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int c = blockIdx.y;
  const int cw = a.head_per_channel ? c : 0;
  const int S = a.S, N = a.N, H = a.H, C = a.C;
  const int NP = ly.npad, NT = NP / 16, ZP = ly.zph, XP = ly.xph;

  __half* z_hi = reinterpret_cast<__half*>(smem + ly.off_zhi);
  __half* z_lo = reinterpret_cast<__half*>(smem + ly.off_zlo);
  __half* x_hi = reinterpret_cast<__half*>(smem + ly.off_xhi);
  __half* x_lo = reinterpret_cast<__half*>(smem + ly.off_xlo);
  float* c_inv = reinterpret_cast<float*>(smem + ly.off_col);   // [NP] 0 past N
  float* c_max = c_inv + NP;                                    // [NP] f_i
  float* c_mu = c_max + NP;                                     // [NP] mu~ (+inf past N)
  float* c_ka = c_mu + NP;                                      // [NP] kappa~
  float* c_nu = c_ka + NP;                                      // [NP] scratch: mu, nu2
  float* c_vm = c_nu + NP;                                      // [NP] raw mu (COMP), 0 past N
  float* c_vk = c_vm + NP;                                      // [NP] raw kappa (COMP)
  float* yred = reinterpret_cast<float*>(smem + ly.off_yred);   // [nwarps][16 MMT][8 NTT]
  float* scr = reinterpret_cast<float*>(smem + ly.off_scr);     // [32]
  float* w1 = scr + 32;   // [32] row sums of W_s + W_t (instance normalisation, see a8)
  const __half* w_hi = reinterpret_cast<const __half*>(
      reinterpret_cast<const unsigned char*>(a.wpack_flash) + (size_t)cw * ly.wpack_bytes);
  const int WLD = 2 * NP;
  const __half* w_lo = w_hi + (16 * MMT) * WLD;
  const float inv_sw = a.wpack_flash_inv_sw[cw];

  // operand tiles start at zero: rows >= N and columns >= S stay zero
  for (int k = tid; k < (ly.off_col - ly.off_zhi) / 16; k += nthr)
    reinterpret_cast<uint4*>(smem + ly.off_zhi)[k] = make_uint4(0, 0, 0, 0);
  if (a.revin) {   // w1[m] = sum_n W_s[m][n] + W_t[m][n] (the head applied to a constant row)
    const float* gs = a.ws + (int64_t)cw * a.M * N;
    const float* gt = a.wt + (int64_t)cw * a.M * N;
    for (int m = tid; m < a.M; m += nthr) {
      float acc = 0.f;
      // (component values: only the trend branch carries the normalised level)
      for (int n = 0; n < N; n++) acc += (COMP ? 0.f : __ldg(gs + m * N + n)) + __ldg(gt + m * N + n);
      w1[m] = acc;
    }
  }
  __syncthreads();

  const int64_t b_begin = (int64_t)blockIdx.x * wins_per_cta;
  int64_t b_end = b_begin + wins_per_cta;
  if (b_end > a.B) b_end = a.B;
  const float half_s = a.half_s;
  for (int64_t b = b_begin; b < b_end; b++) {
    const int64_t series = b * C + c;
    // ---------------- a1: the segmented span is read straight from global memory by the two
    // descriptor passes (the second hits L1/L2): no shared staging, so a 480-segment series
    // fits two CTAs per SM
    const float* xbuf = a.x + b * a.xsb + c * a.xsc + a.r;
    // the next series' span into L2 (one bulk prefetch): the descriptor passes of series b + 1
    // then start from L2 instead of DRAM (16-byte aligned windows; the size rounded down)
    if (tid == 0 && a.x_vec && b + 1 < b_end) {
      const float* nx = xbuf + a.xsb;
      const uint32_t nbytes = (uint32_t)(N * S * 4) & ~15u;
      if (nbytes > 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nx), "r"(nbytes)
                     : "memory");
    }
    // KS >= 2 (S > 16): the descriptor passes with tps threads per segment; S <= 16 keeps one
    // thread per segment (measured: L720/S12 1.18 ms against 1.27-1.39 with the grouped form)
    float sx, sz, mu_r, rr, sr, cmt, ckt;
    int loose;
    if constexpr (KS >= 2) {
      // ---------------- a2: descriptors (Def 4-5), tps threads per segment (the largest power of
      // two <= 8 with N tps <= the CTA's threads and S / tps >= 8): thread r of a segment's group takes t = r, r +
      // tps, .., the segment's sums and maxima by xor shuffles inside the group; the group's
      // leader (r = 0) writes the per-segment scalars.  (Thread per segment left 3/4 of the CTA
      // idle at N = 60 behind three serial S-long passes.)
      // (and >= 8 elements per thread: at S = 12 the group shuffles cost more than they save,
      // measured L720/S12 1.27 vs 1.18 ms with 4 threads per segment)
      int tps = 1;
      while (tps < 8 && N * tps * 2 <= nthr && S >= 16 * tps) tps <<= 1;
      const int gsz = nthr / tps, nl = tid / tps, rr_ = tid - nl * tps;
      auto gsum = [&](float v) {
        for (int o = 1; o < tps; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
      };
      auto gmax = [&](float v) {
        for (int o = 1; o < tps; o <<= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        return v;
      };
      float amx = 0.f, dmx = 0.f;
      for (int base = 0; base < N; base += gsz) {   // CTA-uniform trip count (shuffles)
        const int n = base + nl;
        const bool on = n < N;
        float s1 = 0.f, s3 = 0.f, dm = 0.f;
        if (on) {
          const float* xr = xbuf + n * S;
          const float x0 = xr[0];
          for (int t = rr_; t < S; t += tps) {
            const float d = xr[t] - x0;
            s1 += d;
            s3 = fmaf((float)t - half_s, d, s3);
            amx = fmaxf(amx, fabsf(xr[t]));
            dm = fmaxf(dm, fabsf(d));
          }
        }
        s1 = gsum(s1);
        s3 = gsum(s3);
        dm = gmax(dm);
        if (on) {
          const float ka = s3 * a.inv_v;
          if (rr_ == 0) {
            c_nu[n] = s1 * a.inv_s;          // m1 (mu - x0)
            c_ka[n] = ka;                    // kappa
          }
          // |z| <= 2 max|d|; detrended (metric_variant bit 1): |e| <= |z| + |kappa| (S-1)/2
          dmx = fmaxf(dmx, 2.f * dm + (a.detrend ? fabsf(ka) * half_s : 0.f));
        }
      }
      block_reduce2(amx, dmx, scr, true);
      sx = pow2_scale(amx);
      sz = pow2_scale(dmx);
      // Def 5 in one reduction about the reference m0 = mu_0 (as tc_quad): with d = mu - m0,
      // sum (mu - mubar)^2 = sum d^2 - (sum d)^2 / N
      const float m0 = xbuf[0] + c_nu[0];
      float dsum1 = 0.f, dsum2 = 0.f;
      for (int base = 0; base < N; base += gsz) {
        const int n = base + nl;
        const bool on = n < N;
        float q = 0.f, x0 = 0.f, m1 = 0.f, ka = 0.f;
        if (on) {
          const float* xr = xbuf + n * S;
          x0 = xr[0];
          m1 = c_nu[n];
          ka = c_ka[n];
          const float kd = a.detrend ? ka : 0.f;   // e = z - kappa t~
          for (int t = 2 * rr_; t < S; t += 2 * tps) {   // column pairs (t, t + 1)
            const bool two = t + 1 < S;
            const float v0 = xr[t], v1 = two ? xr[t + 1] : 0.f;
            const float z0 = fmaf(-kd, (float)t - half_s, (v0 - x0) - m1);
            const float z1 = two ? fmaf(-kd, (float)(t + 1) - half_s, (v1 - x0) - m1) : 0.f;
            q = fmaf(z1, z1, fmaf(z0, z0, q));
            store_split_pair(x_hi, x_lo, n * XP + t, v0 * sx, v1 * sx, two);
          }
        }
        q = gsum(q);
        if (on && rr_ == 0) {
          const float mu = x0 + m1;
          c_mu[n] = mu;        // temporarily mu
          c_inv[n] = q;        // temporarily nu2
          // Def 5 uses |z|^2 = |e|^2 + kappa^2 V when the seasonal metric is detrended
          const float nz2 = a.detrend ? fmaf(ka * ka, 1.f / a.inv_v, q) : q;
          const float d = mu - m0;
          dsum1 += d;
          dsum2 += fmaf((float)S * d, d, nz2);
        }
      }
      block_reduce2(dsum1, dsum2, scr, false);
      const float mbar = fmaf(dsum1, a.inv_n, m0);
      const float var = fmaf(-(float)S * dsum1, dsum1 * a.inv_n, dsum2) * a.inv_ns;
      // instance normalisation: descriptors of xhat = (x - mu_r) rr are
      // affine images of those of x; the head runs on x and a8 adds mu_r (1 - w1[m]) + sr b
      mu_r = 0.f, rr = 1.f, sr = 1.f;
      if (a.revin) {
        mu_r = mbar;
        rr = rsqrtf(var + kEpsRevin);
        sr = (var + kEpsRevin) * rr;
      }
      const float inv_var = fast_rcp(fmaf(var * rr, rr, kEpsTrend));   // MUFU, <= ~1 ulp
      cmt = fast_sqrt(inv_var * a.kt) * rr, ckt = cmt * fast_sqrt(a.vtrend);
      // a row whose known bound f_n sits far above its true maximum (between f_n^2 and f_n:
      // a segment with nu^2 not >> eps_s, e.g. constant to within rounding) would leave its
      // largest exponential below 2^-6 at low tau_s, where the fp16 hi/lo split of E loses
      // precision (and below 2^-24 it underflows): such series take exact row maxima (below)
      loose = 0;
      for (int base = 0; base < NP; base += gsz) {
        const int n = base + nl;
        const bool on = n < N;
        float nu2 = 0.f, inv = 0.f, cmu = 0.f, cka = 0.f;
        if (on) {
          nu2 = c_inv[n] * rr * rr;
          inv = rsqrtf(nu2 + kEpsSeasonal);
          cmu = c_mu[n];
          cka = c_ka[n];
          // row-normalised Gram operand Z'_n = z_n rr / sqrt(nu2_n rr^2 + eps_s) (|Z'_n| <= 1):
          // the split keeps ~22 bits relative to every row, and the Gram is rho itself
          const float* xr = xbuf + n * S;
          const float x0 = xr[0], m1 = c_nu[n], q = inv * rr;
          const float kd = a.detrend ? cka : 0.f;
          for (int t = 2 * rr_; t < S; t += 2 * tps) {   // column pairs (t, t + 1)
            const bool two = t + 1 < S;
            const float z0 = fmaf(-kd, (float)t - half_s, (xr[t] - x0) - m1);
            const float z1 = two ? fmaf(-kd, (float)(t + 1) - half_s, (xr[t + 1] - x0) - m1) : 0.f;
            store_split_pair(z_hi, z_lo, n * ZP + t, z0 * q, z1 * q, two);
          }
        }
        __syncwarp();   // the group has read the row's scalars: the leader rewrites them
        if (rr_ == 0 && n < NP) {
          if (on) {
            c_inv[n] = 1.f;                // column factor of rho: 1 (row-normalised Gram)
            c_max[n] = fast_sqrt(nu2) * inv;   // f_n: known row maximum of rho (Cauchy-Schwarz)
            loose |= (c_max[n] - c_max[n] * c_max[n]) * a.ks > 6.f;
            if (COMP) {
              c_vm[n] = cmu;
              c_vk[n] = cka;
            }
            c_mu[n] = (cmu - mu_r) * cmt;
            c_ka[n] = cka * ckt;
          } else {
            c_inv[n] = 0.f;
            c_max[n] = 0.f;
            c_mu[n] = INFINITY;            // exponent -inf: masked key
            c_ka[n] = 0.f;
            if (COMP) c_vm[n] = c_vk[n] = 0.f;
          }
        }
      }
    } else {
      // ---------------- a2: descriptors (Def 4-5), thread per segment
      float amx = 0.f, dmx = 0.f;
      for (int n = tid; n < N; n += nthr) {
        const float* xr = xbuf + n * S;
        const float x0 = xr[0];
        float s1 = 0.f, s3 = 0.f, dm = 0.f;
        for (int t = 0; t < S; t++) {
          const float d = xr[t] - x0;
          s1 += d;
          s3 = fmaf((float)t - half_s, d, s3);
          amx = fmaxf(amx, fabsf(xr[t]));
          dm = fmaxf(dm, fabsf(d));
        }
        c_nu[n] = s1 * a.inv_s;          // m1 (mu - x0)
        c_ka[n] = s3 * a.inv_v;          // kappa
        // |z| <= 2 max|d|; detrended (metric_variant bit 1): |e| <= |z| + |kappa| (S-1)/2
        dmx = fmaxf(dmx, 2.f * dm + (a.detrend ? fabsf(c_ka[n]) * half_s : 0.f));
      }
      block_reduce2(amx, dmx, scr, true);
      sx = pow2_scale(amx);
      sz = pow2_scale(dmx);
      // Def 5 in one reduction about the reference m0 = mu_0 (as tc_quad): with d = mu - m0,
      // sum (mu - mubar)^2 = sum d^2 - (sum d)^2 / N
      const float m0 = xbuf[0] + c_nu[0];
      float dsum1 = 0.f, dsum2 = 0.f;
      for (int n = tid; n < N; n += nthr) {
        const float* xr = xbuf + n * S;
        const float x0 = xr[0], m1 = c_nu[n];
        const float kd = a.detrend ? c_ka[n] : 0.f;   // e = z - kappa t~
        float q = 0.f;
        for (int t = 0; t < S; t += 2) {   // column pairs (t, t + 1)
          const bool two = t + 1 < S;
          const float v0 = xr[t], v1 = two ? xr[t + 1] : 0.f;
          const float z0 = fmaf(-kd, (float)t - half_s, (v0 - x0) - m1);
          const float z1 = two ? fmaf(-kd, (float)(t + 1) - half_s, (v1 - x0) - m1) : 0.f;
          q = fmaf(z1, z1, fmaf(z0, z0, q));
          store_split_pair(x_hi, x_lo, n * XP + t, v0 * sx, v1 * sx, two);
        }
        const float mu = x0 + m1;
        c_mu[n] = mu;        // temporarily mu
        c_inv[n] = q;        // temporarily nu2
        // Def 5 uses |z|^2 = |e|^2 + kappa^2 V when the seasonal metric is detrended
        const float nz2 = a.detrend ? fmaf(c_ka[n] * c_ka[n], 1.f / a.inv_v, q) : q;
        const float d = mu - m0;
        dsum1 += d;
        dsum2 += fmaf((float)S * d, d, nz2);
      }
      block_reduce2(dsum1, dsum2, scr, false);
      const float mbar = fmaf(dsum1, a.inv_n, m0);
      const float var = fmaf(-(float)S * dsum1, dsum1 * a.inv_n, dsum2) * a.inv_ns;
      // instance normalisation: descriptors of xhat = (x - mu_r) rr are
      // affine images of those of x; the head runs on x and a8 adds mu_r (1 - w1[m]) + sr b
      mu_r = 0.f, rr = 1.f, sr = 1.f;
      if (a.revin) {
        mu_r = mbar;
        rr = rsqrtf(var + kEpsRevin);
        sr = (var + kEpsRevin) * rr;
      }
      const float inv_var = fast_rcp(fmaf(var * rr, rr, kEpsTrend));   // MUFU, <= ~1 ulp
      cmt = fast_sqrt(inv_var * a.kt) * rr, ckt = cmt * fast_sqrt(a.vtrend);
      // a row whose known bound f_n sits far above its true maximum (between f_n^2 and f_n:
      // a segment with nu^2 not >> eps_s, e.g. constant to within rounding) would leave its
      // largest exponential below 2^-6 at low tau_s, where the fp16 hi/lo split of E loses
      // precision (and below 2^-24 it underflows): such series take exact row maxima (below)
      loose = 0;
      for (int n = tid; n < NP; n += nthr) {
        if (n < N) {
          const float nu2 = c_inv[n] * rr * rr;
          const float inv = rsqrtf(nu2 + kEpsSeasonal);
          // row-normalised Gram operand Z'_n = z_n rr / sqrt(nu2_n rr^2 + eps_s) (|Z'_n| <= 1):
          // the split keeps ~22 bits relative to every row, and the Gram is rho itself
          {
            const float* xr = xbuf + n * S;
            const float x0 = xr[0], m1 = c_nu[n], q = inv * rr;
            const float kd = a.detrend ? c_ka[n] : 0.f;
            for (int t = 0; t < S; t += 2) {   // column pairs (t, t + 1)
              const bool two = t + 1 < S;
              const float z0 = fmaf(-kd, (float)t - half_s, (xr[t] - x0) - m1);
              const float z1 = two ? fmaf(-kd, (float)(t + 1) - half_s, (xr[t + 1] - x0) - m1) : 0.f;
              store_split_pair(z_hi, z_lo, n * ZP + t, z0 * q, z1 * q, two);
            }
          }
          c_inv[n] = 1.f;                // column factor of rho: 1 (row-normalised Gram)
          c_max[n] = fast_sqrt(nu2) * inv;   // f_n: known row maximum of rho (Cauchy-Schwarz)
          loose |= (c_max[n] - c_max[n] * c_max[n]) * a.ks > 6.f;
          if (COMP) {
            c_vm[n] = c_mu[n];
            c_vk[n] = c_ka[n];
          }
          c_mu[n] = (c_mu[n] - mu_r) * cmt;
          c_ka[n] = c_ka[n] * ckt;
        } else {
          c_inv[n] = 0.f;
          c_max[n] = 0.f;
          c_mu[n] = INFINITY;            // exponent -inf: masked key
          c_ka[n] = 0.f;
          if (COMP) c_vm[n] = c_vk[n] = 0.f;
        }
      }
    }
    loose = __syncthreads_or(loose);

    // (KS <= 3: one chunk, compile-time, so the loop and the offsets fold away)
    const int nch = KS >= 4 ? ly.nch : 1;
    for (int tc = 0; tc < nch; tc++) {
    const int tb = KS >= 4 ? tc * NTT : 0;   // first t tile of this chunk
    // ---------------- a3..a7 per 16-row query tile
    float yacc[MMT][NTT][4];
#pragma unroll
    for (int mm = 0; mm < MMT; mm++)
#pragma unroll
      for (int nt = 0; nt < NTT; nt++)
#pragma unroll
        for (int e = 0; e < 4; e++) yacc[mm][nt][e] = 0.f;
    const float rsz2 = a.ks;   // the Gram of the row-normalised Z' is rho
    for (int qt = warp; qt < NT; qt += nwarps) {
      uint32_t zah[KS][4], zal[KS][4];
#pragma unroll
      for (int ks = 0; ks < KS; ks++) {
        const int off = (16 * qt + (lane & 7) + 8 * (q8 & 1)) * ZP + 16 * ks + 8 * (q8 >> 1);
        ldsm_x4(zah[ks], z_hi + off);
        ldsm_x4(zal[ks], z_lo + off);
      }
      float rk[2], nb[2], mi[2], ki[2];
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int ii = 16 * qt + 8 * h + gq;
        rk[h] = (ii < N ? c_inv[ii] : 1.f) * rsz2;
        nb[h] = -c_max[ii] * a.ks;
        mi[h] = ii < N ? c_mu[ii] : 0.f;
        ki[h] = c_ka[ii];
      }
      if (loose) {
        // exact row maxima of rho over the key tiles (a Gram-only pass; CTA-uniform branch,
        // taken only by series with a loose bound) as the softmax shift
        float rmx[2] = {-INFINITY, -INFINITY};
        for (int jt = 0; jt < NT; jt++) {
          float g[2][4];
#pragma unroll
          for (int nt = 0; nt < 2; nt++)
#pragma unroll
            for (int e = 0; e < 4; e++) g[nt][e] = 0.f;
#pragma unroll
          for (int ks = 0; ks < KS; ks++) {
            uint32_t bh[4], bl[4];
            const int off = (16 * jt + (lane & 7) + 8 * (q8 >> 1)) * ZP + 16 * ks + 8 * (q8 & 1);
            ldsm_x4(bh, z_hi + off);
            ldsm_x4(bl, z_lo + off);
            mma16816(g[0], zal[ks], bh[0], bh[1]);
            mma16816(g[1], zal[ks], bh[2], bh[3]);
            mma16816(g[0], zah[ks], bl[0], bl[1]);
            mma16816(g[1], zah[ks], bl[2], bl[3]);
            mma16816(g[0], zah[ks], bh[0], bh[1]);
            mma16816(g[1], zah[ks], bh[2], bh[3]);
          }
#pragma unroll
          for (int nt = 0; nt < 2; nt++) {
            const int j = 16 * jt + 8 * nt + 2 * cq;
#pragma unroll
            for (int h = 0; h < 2; h++) {
              if (j < N) rmx[h] = fmaxf(rmx[h], g[nt][2 * h]);
              if (j + 1 < N) rmx[h] = fmaxf(rmx[h], g[nt][2 * h + 1]);
            }
          }
        }
#pragma unroll
        for (int h = 0; h < 2; h++) {
          rmx[h] = fmaxf(rmx[h], __shfl_xor_sync(0xffffffffu, rmx[h], 1));
          rmx[h] = fmaxf(rmx[h], __shfl_xor_sync(0xffffffffu, rmx[h], 2));
          const int ii = 16 * qt + 8 * h + gq;
          if (ii < N) nb[h] = -rmx[h] * rk[h];   // c_inv = 1: the Gram is rho itself
        }
      }
      float as_[NTT][4], at_[NTT][4];
#pragma unroll
      for (int nt = 0; nt < NTT; nt++)
#pragma unroll
        for (int e = 0; e < 4; e++) as_[nt][e] = at_[nt][e] = 0.f;
      float ssum[2] = {0.f, 0.f}, tsum[2] = {0.f, 0.f};
      // COMP: sum_j E_ij mu_j, E_ij kappa_j for both branches (raw descriptors)
      float csm[2] = {0.f, 0.f}, csk[2] = {0.f, 0.f}, ctm[2] = {0.f, 0.f}, ctk[2] = {0.f, 0.f};

      for (int jt = 0; jt < NT; jt++) {
        // a3: Gram tile (16 query rows x 16 keys)
        float g[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; nt++)
#pragma unroll
          for (int e = 0; e < 4; e++) g[nt][e] = 0.f;
#pragma unroll
        for (int ks = 0; ks < KS; ks++) {
          uint32_t bh[4], bl[4];
          const int off = (16 * jt + (lane & 7) + 8 * (q8 >> 1)) * ZP + 16 * ks + 8 * (q8 & 1);
          ldsm_x4(bh, z_hi + off);
          ldsm_x4(bl, z_lo + off);
          mma16816(g[0], zal[ks], bh[0], bh[1]);
          mma16816(g[1], zal[ks], bh[2], bh[3]);
          mma16816(g[0], zah[ks], bl[0], bl[1]);
          mma16816(g[1], zah[ks], bl[2], bl[3]);
          mma16816(g[0], zah[ks], bh[0], bh[1]);
          mma16816(g[1], zah[ks], bh[2], bh[3]);
        }
        // a4/a5: exponentials with known maxima, row sums, E as A fragments (hi/lo)
        uint32_t esh[4], esl[4], eth[4], etl[4];
#pragma unroll
        for (int nt = 0; nt < 2; nt++) {
          const int j = 16 * jt + 8 * nt + 2 * cq;
          const float2 cinv = *reinterpret_cast<const float2*>(c_inv + j);
          const float2 cmu = *reinterpret_cast<const float2*>(c_mu + j);
          const float2 cka = *reinterpret_cast<const float2*>(c_ka + j);
          float2 vm = f2(0.f), vk = f2(0.f);
          if (COMP) {
            vm = *reinterpret_cast<const float2*>(c_vm + j);
            vk = *reinterpret_cast<const float2*>(c_vk + j);
          }
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const float2 u = mul2(make_float2(g[nt][2 * h], g[nt][2 * h + 1]), cinv);
            const float2 arg = fma2(u, f2(rk[h]), f2(nb[h]));
            float2 es = make_float2(fast_ex2(arg.x), fast_ex2(arg.y));
            if (j >= N) es.x = 0.f;
            if (j + 1 >= N) es.y = 0.f;
            const float2 dm = add2(f2(mi[h]), make_float2(-cmu.x, -cmu.y));
            const float2 dk = add2(f2(ki[h]), make_float2(-cka.x, -cka.y));
            const float2 ea = fma2(make_float2(-dk.x, -dk.y), dk, mul2(make_float2(-dm.x, -dm.y), dm));
            const float2 et = make_float2(fast_ex2(ea.x), fast_ex2(ea.y));
            ssum[h] += es.x + es.y;
            tsum[h] += et.x + et.y;
            if (COMP) {
              csm[h] = fmaf(es.x, vm.x, fmaf(es.y, vm.y, csm[h]));
              csk[h] = fmaf(es.x, vk.x, fmaf(es.y, vk.y, csk[h]));
              ctm[h] = fmaf(et.x, vm.x, fmaf(et.y, vm.y, ctm[h]));
              ctk[h] = fmaf(et.x, vk.x, fmaf(et.y, vk.y, ctk[h]));
            }
            // A fragment register index: a0 (h0, nt0), a1 (h1, nt0), a2 (h0, nt1), a3 (h1, nt1)
            split2(es, esh[2 * nt + h], esl[2 * nt + h]);
            split2(et, eth[2 * nt + h], etl[2 * nt + h]);
          }
        }
        // a6: P += E X_j  (X_j rows of this key tile, t tiles)
#pragma unroll
        for (int tp = 0; tp < (NTT + 1) / 2; tp++) {
          uint32_t xh[4], xl[4];
          const int krow = 16 * jt + (lane & 7) + 8 * (q8 & 1);
          if (2 * tp + 1 < NTT) {
            const int off = krow * XP + 8 * (tb + 2 * tp + (q8 >> 1));
            ldsm_x4_t(xh, x_hi + off);
            ldsm_x4_t(xl, x_lo + off);
          } else {
            const int off = krow * XP + 8 * (tb + 2 * tp);
            ldsm_x2_t(xh[0], xh[1], x_hi + off);
            ldsm_x2_t(xl[0], xl[1], x_lo + off);
          }
#pragma unroll
          for (int u2 = 0; u2 < 2; u2++) {
            const int nt = 2 * tp + u2;
            if (nt < NTT) {
              mma16816(as_[nt], esl, xh[2 * u2], xh[2 * u2 + 1]);
              if constexpr (!COMP) mma16816(at_[nt], etl, xh[2 * u2], xh[2 * u2 + 1]);
              mma16816(as_[nt], esh, xl[2 * u2], xl[2 * u2 + 1]);
              if constexpr (!COMP) mma16816(at_[nt], eth, xl[2 * u2], xl[2 * u2 + 1]);
              mma16816(as_[nt], esh, xh[2 * u2], xh[2 * u2 + 1]);
              if constexpr (!COMP) mma16816(at_[nt], eth, xh[2 * u2], xh[2 * u2 + 1]);
            }
          }
        }
      }
      // row sums over the quad, normalise: P rows of this tile
#pragma unroll
      for (int h = 0; h < 2; h++) {
        ssum[h] += __shfl_xor_sync(0xffffffffu, ssum[h], 1);
        ssum[h] += __shfl_xor_sync(0xffffffffu, ssum[h], 2);
        tsum[h] += __shfl_xor_sync(0xffffffffu, tsum[h], 1);
        tsum[h] += __shfl_xor_sync(0xffffffffu, tsum[h], 2);
        const int ii = 16 * qt + 8 * h + gq;
        ssum[h] = ii < N ? fast_rcp(ssum[h]) : 0.f;   // row sums >= the largest term (normal)
        tsum[h] = ii < N ? fast_rcp(tsum[h]) : 0.f;
        if (COMP) {
#pragma unroll
          for (int o = 1; o <= 2; o <<= 1) {
            csm[h] += __shfl_xor_sync(0xffffffffu, csm[h], o);
            csk[h] += __shfl_xor_sync(0xffffffffu, csk[h], o);
            ctm[h] += __shfl_xor_sync(0xffffffffu, ctm[h], o);
            ctk[h] += __shfl_xor_sync(0xffffffffu, ctk[h], o);
          }
          // in the X' = x sx units of the accumulators; d1 = bit 1, d0 = 1 - bit 0
          csm[h] *= ssum[h] * sx;
          csk[h] *= ssum[h] * sx * (a.detrend ? 1.f : 0.f);
          ctm[h] *= tsum[h] * sx;
          ctk[h] *= tsum[h] * sx * (a.vtrend != 0.f ? 1.f : 0.f);
        }
      }
      // a7: P fragments -> B operand (k = i, n = t) via movmatrix; Y += W'_s P_s + W'_t P_t
      uint32_t psh[NTT][2], psl[NTT][2], pth[NTT][2], ptl[NTT][2];
#pragma unroll
      for (int nt = 0; nt < NTT; nt++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          uint32_t hi, lo;
          float2 ps = mul2(make_float2(as_[nt][2 * h], as_[nt][2 * h + 1]), f2(ssum[h]));
          float2 pt = mul2(make_float2(at_[nt][2 * h], at_[nt][2 * h + 1]), f2(tsum[h]));
          if (COMP) {   // component values: subtract / substitute the rank-2 parts
            const float t0 = (float)(8 * (tb + nt) + 2 * cq) - half_s;
            const float2 tt = make_float2(t0, t0 + 1.f);
            ps = add2(ps, make_float2(-fmaf(csk[h], tt.x, csm[h]), -fmaf(csk[h], tt.y, csm[h])));
            pt = make_float2(fmaf(ctk[h], tt.x, ctm[h]), fmaf(ctk[h], tt.y, ctm[h]));
          }
          split2(ps, hi, lo);
          psh[nt][h] = movm_t(hi);
          psl[nt][h] = movm_t(lo);
          split2(pt, hi, lo);
          pth[nt][h] = movm_t(hi);
          ptl[nt][h] = movm_t(lo);
        }
#pragma unroll
      for (int mm = 0; mm < MMT; mm++) {
        uint32_t wsh[4], wsl[4], wth[4], wtl[4];
        ldg_afrag(w_hi, WLD, 16 * mm, 16 * qt, lane, wsh);
        ldg_afrag(w_lo, WLD, 16 * mm, 16 * qt, lane, wsl);
        ldg_afrag(w_hi, WLD, 16 * mm, NP + 16 * qt, lane, wth);
        ldg_afrag(w_lo, WLD, 16 * mm, NP + 16 * qt, lane, wtl);
#pragma unroll
        for (int nt = 0; nt < NTT; nt++) {
          mma16816(yacc[mm][nt], wsl, psh[nt][0], psh[nt][1]);
          mma16816(yacc[mm][nt], wsh, psl[nt][0], psl[nt][1]);
          mma16816(yacc[mm][nt], wsh, psh[nt][0], psh[nt][1]);
          mma16816(yacc[mm][nt], wtl, pth[nt][0], pth[nt][1]);
          mma16816(yacc[mm][nt], wth, ptl[nt][0], ptl[nt][1]);
          mma16816(yacc[mm][nt], wth, pth[nt][0], pth[nt][1]);
        }
      }
    }
    // ---------------- a8: fixed-order reduction over warps, scale, bias, store
    {
      constexpr int YR = 8 * NTT;
      float* yw = yred + warp * (16 * MMT) * YR;
#pragma unroll
      for (int mm = 0; mm < MMT; mm++)
#pragma unroll
        for (int nt = 0; nt < NTT; nt++)
#pragma unroll
          for (int h = 0; h < 2; h++)
            *reinterpret_cast<float2*>(yw + (16 * mm + 8 * h + gq) * YR + 8 * nt + 2 * cq) =
                make_float2(yacc[mm][nt][2 * h], yacc[mm][nt][2 * h + 1]);
      __syncthreads();
      const float ysc = inv_sw / sx;
      const float* gb = a.bias + (int64_t)cw * H;
      float* yg = a.y + series * H;
      for (int h = tid; h < H; h += nthr) {
        const int m = h / S, t = h - m * S - 8 * tb;
        if (t < 0 || t >= YR) continue;   // another chunk's columns
        float v = 0.f;
        for (int w = 0; w < nwarps; w++) v += yred[(w * (16 * MMT) + m) * YR + t];
        yg[h] = a.revin ? v * ysc + fmaf(__ldg(gb + h), sr, mu_r * (1.f - w1[m]))
                        : v * ysc + __ldg(gb + h);
      }
      __syncthreads();
    }
    }   // t chunks
  }
}

bool plan_flash_kernel(const FwdArgs& a, int max_smem_optin, FlashPlan* p) {
  if (a.N <= 16 || a.N > 512 || a.M > 32 || a.S > 96) return false;
  FlashLayout& ly = p->ly;
  p->ks = (a.S + 15) / 16;
  p->ntt = (a.S + 7) / 8;
  if (p->ntt == 5) p->ntt = 6;
  if (p->ntt == 1) p->ntt = 2;
  ly.nch = 1;
  if (a.S > 48) {   // chunks of 4 (S <= 64) or 6 (S <= 96) t tiles
    p->ks = a.S <= 64 ? 4 : 6;
    ly.nch = 2;
    p->ntt = (((a.S + 7) / 8) + 1) / 2;
    p->ntt = p->ntt <= 4 ? 4 : 6;
  }
  p->mmt = a.M <= 16 ? 1 : 2;
  ly.npad = flash_npad(a.N);
  auto odd8 = [](int v) { v = (v + 7) & ~7; if (((v / 8) & 1) == 0) v += 8; return v; };
  ly.zph = odd8(16 * p->ks);
  ly.xph = odd8(8 * p->ntt * ly.nch);   // whole chunks (zero columns past S)
  int off = 0;   // (no fp32 staging of the series: the descriptor passes read global memory)
  ly.off_zhi = off;
  off += ly.npad * ly.zph * 2;
  ly.off_zlo = off;
  off += ly.npad * ly.zph * 2;
  ly.off_xhi = off;
  off += ly.npad * ly.xph * 2;
  ly.off_xlo = off;
  off += ly.npad * ly.xph * 2;
  off = (off + 15) & ~15;
  ly.off_col = off;
  off += 7 * ly.npad * 4;   // c_inv, c_max, c_mu, c_ka, c_nu, c_vm, c_vk
  off = (off + 15) & ~15;
  ly.off_yred = off;
  // one warp per 16-row query tile, up to 8: short series (N <= 64) run 4-warp CTAs so
  // two of them share an SM instead of leaving half an 8-warp CTA idle
  const int nt = ly.npad / 16;
  p->warps = nt >= 8 ? 8 : (nt >= 4 ? 4 : 2);
  off += p->warps * (16 * p->mmt) * (8 * p->ntt) * 4;
  ly.off_scr = off;
  off += 64 * 4;   // block-reduce scratch [32] + w1 [32]
  p->smem_bytes = (size_t)((off + 127) & ~127);
  ly.wpack_bytes = flash_wpack_bytes(a.N, a.M);
  if (p->smem_bytes > (size_t)max_smem_optin) return false;
  p->wins_per_cta = 4;
  return true;
}

template <int KS, int NTT, int MMT, bool COMP>
static cudaError_t launch_flash_t(const FwdArgs& a, const FlashPlan& p, cudaStream_t st) {
  auto k = prnet_fwd_flash_kernel<KS, NTT, MMT, COMP>;
  cudaError_t e =
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((a.B + p.wins_per_cta - 1) / p.wins_per_cta), (unsigned)a.C);
  k<<<grid, 32 * p.warps, p.smem_bytes, st>>>(a, p.ly, p.wins_per_cta);
  return cudaGetLastError();
}

template <int KS, int NTT>
static cudaError_t launch_flash_m(const FwdArgs& a, const FlashPlan& p, cudaStream_t st) {
  if (a.comp)
    return p.mmt == 1 ? launch_flash_t<KS, NTT, 1, true>(a, p, st)
                      : launch_flash_t<KS, NTT, 2, true>(a, p, st);
  return p.mmt == 1 ? launch_flash_t<KS, NTT, 1, false>(a, p, st)
                    : launch_flash_t<KS, NTT, 2, false>(a, p, st);
}

cudaError_t launch_flash_kernel(const FwdArgs& a, const FlashPlan& p, cudaStream_t st) {
  switch (p.ks * 10 + p.ntt) {
    case 12: return launch_flash_m<1, 2>(a, p, st);   // S <= 16
    case 23: return launch_flash_m<2, 3>(a, p, st);   // S in (16, 24]
    case 24: return launch_flash_m<2, 4>(a, p, st);   // S in (24, 32]
    case 36: return launch_flash_m<3, 6>(a, p, st);   // S in (32, 48]
    case 44: return launch_flash_m<4, 4>(a, p, st);   // S in (48, 64], 2 chunks
    case 66: return launch_flash_m<6, 6>(a, p, st);   // S in (64, 96], 2 chunks
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace prnet
