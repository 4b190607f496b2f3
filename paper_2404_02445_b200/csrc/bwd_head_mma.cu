// bwd_head_mma.cu -- backward pass of the PRNet head on the tensor cores (SURVEY §8(f) f4,
// reading R-f6 in DESIGN.md §3), for N <= 32, M <= 32, S in {8, 16, 24, 32} and the plain
// reading (the level-only trend included; the detrended metric and instance normalisation
// stay on bwd_head.cu's FP32 kernel):
//   dW_s[m][n] = sum_{series, t} dY[m][t] P_s[n][t],  dW_t likewise,  db[h] = sum dy[h],
// with P = A X the patterns of the forward (Def 9), recomputed per series.
//
// bwd_head.cu's FP32 kernel broadcasts every row of X, Z and dY from shared memory to all
// lanes (one 128-bit broadcast = 4 LSU wavefronts per 4 values): ~2300 wavefronts per series,
// 28 ms on Traffic.  Here every contraction is an mma.sync m16n8k16 (m16n8k8 for an S tail) in
// split fp16 (v = hi + lo, products hh + hl + lh, fp32 accumulation: DESIGN.md §6), operands
// from shared memory by ldmatrix or straight from the previous product's accumulators:
//   Gram   rho = Zhat Zhat^T           A, B = Zhat rows (ldmatrix), Zhat = z / sqrt(nu2 + eps_s)
//   softmax on the Gram accumulators   exact row maxima (quad shuffles), trend logits from the
//                                      shuffled descriptors, rows normalised in registers
//   P' = A X'                          A from the softmax accumulators (the C layout of two
//                                      n-tiles is the A layout of one k-step), X' = x sx by
//                                      ldmatrix.trans
//   G = dY' P'^T                       A = dY' = dY sy rows (ldmatrix), B from P's accumulators
//                                      (row n of P = column n of the B tile: no transposition)
//   dW += G / (sx sy)                  FP32, in registers over all series of the warp
// sx, sy are exact powers of two per series (|X'|, |dY'| < 1, so every fp16 split is in range
// and |P'| <= 1).  One warp per series, 8 warps per CTA, one channel per CTA; the warps' dW are
// reduced in a fixed order into one partial per CTA (the FP32 kernel's partial layout), then
// prnet_bwd_reduce sums the partials in fp64.  Deterministic, no atomics.
#include "prnet_internal.cuh"
#include "mma_common.cuh"

namespace prnet {

namespace {

constexpr int kBmWarps = 4;
constexpr int kBmMinBlocks = 3;   // 12 warps per SM: <= 168 registers

// split a pair into (hi, lo) f16x2 registers (mma_common.cuh's split2)
__device__ __forceinline__ void split_pair(float a, float b, uint32_t& hi, uint32_t& lo) {
  split2(make_float2(a, b), hi, lo);
}
// hh + hl + lh with fp32 accumulation, m16n8k16
__device__ __forceinline__ void mma3(float (&c)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4],
                                     uint32_t bh0, uint32_t bh1, uint32_t bl0, uint32_t bl1) {
  mma16816_nv(c, al, bh0, bh1);
  mma16816_nv(c, ah, bl0, bl1);
  mma16816_nv(c, ah, bh0, bh1);
}
// m16n8k8
__device__ __forceinline__ void mma3k8(float (&c)[4], uint32_t ah0, uint32_t ah1, uint32_t al0,
                                       uint32_t al1, uint32_t bh, uint32_t bl) {
  mma1688_nv(c, al0, al1, bh);
  mma1688_nv(c, ah0, ah1, bl);
  mma1688_nv(c, ah0, ah1, bh);
}

}  // namespace

// PB: bytes per fp16 row of the [row][t] operand tiles: 2S, + 16 when S / 8 is even, so a row
// is an odd number of 16-byte units and the 8 rows of an ldmatrix 8x8 block hit 8 different
// bank groups
template <int S>
struct BmCfg {
  static constexpr int KT = S / 8;                        // 8-wide t tiles
  static constexpr int PB = (KT & 1) ? 2 * S : 2 * S + 16;
  static constexpr int TILE = 32 * PB;                    // one 32-row tile
  static constexpr int PER_WARP_TILES = 6 * TILE;         // Z hi/lo, X hi/lo, dY hi/lo
  // the bias gradient [H] after both the tiles and the final [2][32][32] fp32 reduction area
  static constexpr int OFF_DB = PER_WARP_TILES > 8192 ? PER_WARP_TILES : 8192;
};

template <int S>
__global__ void __launch_bounds__(32 * kBmWarps, kBmMinBlocks) prnet_bwd_head_mma_kernel(FwdArgs a, const float* __restrict__ dy,
                                                                           float* __restrict__ part,
                                                                           int wins_per_cta, int per_warp) {
  using K = BmCfg<S>;
  constexpr int KT = K::KT, PB = K::PB;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.y, C = a.C;
  const int N = a.N, M = a.M, H = a.H;
  const int g = lane >> 2, q = lane & 3;
  unsigned char* wb = smem + (size_t)warp * per_warp;
  unsigned char* Zh = wb;
  unsigned char* Zl = Zh + K::TILE;
  unsigned char* Xh = Zl + K::TILE;
  unsigned char* Xl = Xh + K::TILE;
  unsigned char* Yh = Xl + K::TILE;
  unsigned char* Yl = Yh + K::TILE;
  float* accB = reinterpret_cast<float*>(wb + K::OFF_DB);   // [H] bias gradient
  for (int k = lane; k < H; k += 32) accB[k] = 0.f;

  // dW_s, dW_t accumulators: [branch][m-tile][n-tile][4], element (m = 16 mt + g + 8 (r / 2),
  // n = 8 nt + 2 q + (r & 1))
  float acc[2][2][4][4];
#pragma unroll
  for (int br = 0; br < 2; br++)
#pragma unroll
    for (int mt = 0; mt < 2; mt++)
#pragma unroll
      for (int nt = 0; nt < 4; nt++)
#pragma unroll
        for (int r = 0; r < 4; r++) acc[br][mt][nt][r] = 0.f;

  // column masks of the logits (0 or -inf): j = 8 nt + 2 q + u < N
  float cneg[4][2];
#pragma unroll
  for (int nt = 0; nt < 4; nt++)
#pragma unroll
    for (int u = 0; u < 2; u++) cneg[nt][u] = 8 * nt + 2 * q + u < N ? 0.f : -INFINITY;
  const int i = lane;
  const bool xvec = a.x_vec != 0;
  const bool yvec = (H & 3) == 0 && (((uintptr_t)dy) & 15u) == 0;
  const int64_t b0 = (int64_t)blockIdx.x * wins_per_cta;
  const int64_t b1 = min(b0 + (int64_t)wins_per_cta, a.B);
  for (int64_t b = b0 + warp; b < b1; b += kBmWarps) {
    const int64_t series = b * C + c;
    // ---------------- a1: lane i <- segment row i, lane m <- dY row m (0 past H)
    float xv[S], dv[S];
    {
      const float* xg = a.x + b * a.xsb + c * a.xsc + a.r + (int64_t)i * S;
#pragma unroll
      for (int t = 0; t < S; t += 4) {
        if (i < N) {
          if (xvec) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(xg + t));
            xv[t] = v.x; xv[t + 1] = v.y; xv[t + 2] = v.z; xv[t + 3] = v.w;
          } else {
#pragma unroll
            for (int u = 0; u < 4; u++) xv[t + u] = __ldg(xg + t + u);
          }
        } else {
#pragma unroll
          for (int u = 0; u < 4; u++) xv[t + u] = 0.f;
        }
      }
      const float* yg = dy + series * H + (int64_t)i * S;
      const int hb = i * S;
#pragma unroll
      for (int t = 0; t < S; t += 4) {
        if (i < M && yvec && hb + t + 3 < H) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(yg + t));
          dv[t] = v.x; dv[t + 1] = v.y; dv[t + 2] = v.z; dv[t + 3] = v.w;
        } else {
#pragma unroll
          for (int u = 0; u < 4; u++) dv[t + u] = (i < M && hb + t + u < H) ? __ldg(yg + t + u) : 0.f;
        }
      }
    }
    // ---------------- a2: descriptors (Def 3-5) from d = x - x0
    const bool valid = i < N;
    const float x0 = xv[0];
    float s1 = 0.f, s3 = 0.f;
#pragma unroll
    for (int t = 0; t < S; t++) {
      const float d = xv[t] - x0;
      s1 += d;
      s3 = fmaf((float)t - a.half_s, d, s3);
    }
    const float m1 = s1 * a.inv_s, mu = x0 + m1, kap = s3 * a.inv_v;
    float zv[S];
    float nu2 = 0.f;
#pragma unroll
    for (int t = 0; t < S; t++) {
      zv[t] = valid ? (xv[t] - x0) - m1 : 0.f;
      nu2 = fmaf(zv[t], zv[t], nu2);
    }
    const float mbar = warp_sum(valid ? mu : 0.f) * a.inv_n;
    const float var = warp_sum(valid ? nu2 + (float)S * (mu - mbar) * (mu - mbar) : 0.f) * a.inv_ns;
    // series-level factors by MUFU reciprocal / square root (<= ~1 ulp), as the forward kernels
    const float inv_var = fast_rcp(var + kEpsTrend);
    const float tsc = fast_sqrt(inv_var * a.kt);
    const float mtc = mu * tsc, ktc = kap * (tsc * fast_sqrt(a.vtrend));
    const float zsc = valid ? rsqrtf(nu2 + kEpsSeasonal) : 0.f;
    // exact power-of-two scales: |X'| = |x sx| < 1, |dY'| = |dy sy| < 1
    float mx = 0.f, my = 0.f;
#pragma unroll
    for (int t = 0; t < S; t++) {
      mx = fmaxf(mx, fabsf(xv[t]));
      my = fmaxf(my, fabsf(dv[t]));
    }
    const float sx = pow2_scale(warp_max_nonneg(mx)), sy = pow2_scale(warp_max_nonneg(my));
    // ---------------- operand rows (fp16 hi / lo): Zhat, X', dY' (row = lane)
    __syncwarp();   // the previous series' tiles are read
    {
      unsigned char* zr = Zh + lane * PB;
      unsigned char* xr = Xh + lane * PB;
      unsigned char* yr = Yh + lane * PB;
#pragma unroll
      for (int t = 0; t < S; t += 8) {
        uint4 h, l;
        split_pair(zv[t] * zsc, zv[t + 1] * zsc, h.x, l.x);
        split_pair(zv[t + 2] * zsc, zv[t + 3] * zsc, h.y, l.y);
        split_pair(zv[t + 4] * zsc, zv[t + 5] * zsc, h.z, l.z);
        split_pair(zv[t + 6] * zsc, zv[t + 7] * zsc, h.w, l.w);
        *reinterpret_cast<uint4*>(zr + 2 * t) = h;
        *reinterpret_cast<uint4*>(zr + K::TILE + 2 * t) = l;
        split_pair(xv[t] * sx, xv[t + 1] * sx, h.x, l.x);
        split_pair(xv[t + 2] * sx, xv[t + 3] * sx, h.y, l.y);
        split_pair(xv[t + 4] * sx, xv[t + 5] * sx, h.z, l.z);
        split_pair(xv[t + 6] * sx, xv[t + 7] * sx, h.w, l.w);
        *reinterpret_cast<uint4*>(xr + 2 * t) = h;
        *reinterpret_cast<uint4*>(xr + K::TILE + 2 * t) = l;
        split_pair(dv[t] * sy, dv[t + 1] * sy, h.x, l.x);
        split_pair(dv[t + 2] * sy, dv[t + 3] * sy, h.y, l.y);
        split_pair(dv[t + 4] * sy, dv[t + 5] * sy, h.z, l.z);
        split_pair(dv[t + 6] * sy, dv[t + 7] * sy, h.w, l.w);
        *reinterpret_cast<uint4*>(yr + 2 * t) = h;
        *reinterpret_cast<uint4*>(yr + K::TILE + 2 * t) = l;
      }
    }
    // bias gradient: db[h] += dy[h] (L1-resident re-read)
    for (int k = lane; k < H; k += 32) accB[k] += __ldg(dy + series * H + k);
    __syncwarp();

    // ---------------- a3: Gram rho = Zhat Zhat^T, 32 x 32 in two m-tiles x four n-tiles
    float gacc[2][4][4];
#pragma unroll
    for (int mt = 0; mt < 2; mt++)
#pragma unroll
      for (int nt = 0; nt < 4; nt++)
#pragma unroll
        for (int r = 0; r < 4; r++) gacc[mt][nt][r] = 0.f;
#pragma unroll
    for (int kk = 0; kk < KT / 2; kk++) {   // k16 steps
      const int t0 = 16 * kk;
      uint32_t ah[2][4], al[2][4];
#pragma unroll
      for (int mt = 0; mt < 2; mt++) {
        const unsigned char* p = Zh + (16 * mt + (lane & 15)) * PB + 2 * (t0 + 8 * (lane >> 4));
        ldsm_x4(ah[mt], p);
        ldsm_x4(al[mt], p + K::TILE);
      }
#pragma unroll
      for (int np = 0; np < 2; np++) {   // pairs of n-tiles: x4 = (nt, k lo), (nt, k hi), (nt+1, ..)
        uint32_t bh[4], bl[4];
        const unsigned char* p =
            Zh + (16 * np + (lane & 7) + 8 * (lane >> 4)) * PB + 2 * (t0 + 8 * ((lane >> 3) & 1));
        ldsm_x4(bh, p);
        ldsm_x4(bl, p + K::TILE);
#pragma unroll
        for (int mt = 0; mt < 2; mt++) {
          mma3(gacc[mt][2 * np], ah[mt], al[mt], bh[0], bh[1], bl[0], bl[1]);
          mma3(gacc[mt][2 * np + 1], ah[mt], al[mt], bh[2], bh[3], bl[2], bl[3]);
        }
      }
    }
    if constexpr (KT & 1) {   // k8 tail: t in [S - 8, S)
      const int t0 = S - 8;
      uint32_t ah[2][2], al[2][2];
#pragma unroll
      for (int mt = 0; mt < 2; mt++) {
        const unsigned char* p = Zh + (16 * mt + (lane & 15)) * PB + 2 * t0;
        ldsm_x2(ah[mt][0], ah[mt][1], p);
        ldsm_x2(al[mt][0], al[mt][1], p + K::TILE);
      }
      {   // x4 = the four n-tiles' 8 x 8 blocks at k = t0
        uint32_t bh[4], bl[4];
        const unsigned char* p = Zh + (8 * (lane >> 3) + (lane & 7)) * PB + 2 * t0;
        ldsm_x4(bh, p);
        ldsm_x4(bl, p + K::TILE);
#pragma unroll
        for (int mt = 0; mt < 2; mt++)
#pragma unroll
          for (int nt = 0; nt < 4; nt++)
            mma3k8(gacc[mt][nt], ah[mt][0], ah[mt][1], al[mt][0], al[mt][1], bh[nt], bl[nt]);
      }
    }

    // ---------------- a4 + a5: both softmaxes on the accumulator layout; P' = A X' per branch
    // descriptors of the columns j = 8 nt + 2 q + e and of the rows i = 16 mt + g + 8 h
    float cmt[4][2], ckt[4][2], rmt[2][2], rkt[2][2];
#pragma unroll
    for (int nt = 0; nt < 4; nt++)
#pragma unroll
      for (int e = 0; e < 2; e++) {
        cmt[nt][e] = __shfl_sync(0xffffffffu, mtc, 8 * nt + 2 * q + e);
        ckt[nt][e] = __shfl_sync(0xffffffffu, ktc, 8 * nt + 2 * q + e);
      }
#pragma unroll
    for (int mt = 0; mt < 2; mt++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        rmt[mt][h] = __shfl_sync(0xffffffffu, mtc, 16 * mt + g + 8 * h);
        rkt[mt][h] = __shfl_sync(0xffffffffu, ktc, 16 * mt + g + 8 * h);
      }
    // per branch: softmax -> P' = A X' -> G = dY' P'^T -> dW += G / (sx sy) (one branch's
    // patterns live at a time)
    const float gsc = 1.f / (sx * sy);   // exact (powers of two)
#pragma unroll
    for (int br = 0; br < 2; br++) {
      float e[2][4][4];
#pragma unroll
      for (int mt = 0; mt < 2; mt++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int row = 16 * mt + g + 8 * h;
          float lg[4][2];
          float rmax = -INFINITY;
#pragma unroll
          for (int nt = 0; nt < 4; nt++)
#pragma unroll
            for (int u = 0; u < 2; u++) {
              float v;
              if (br == 0) {
                v = fmaf(gacc[mt][nt][2 * h + u], a.ks, cneg[nt][u]);
              } else {
                const float dm = rmt[mt][h] - cmt[nt][u], dk = rkt[mt][h] - ckt[nt][u];
                v = cneg[nt][u] - fmaf(dm, dm, dk * dk);
              }
              lg[nt][u] = v;
              rmax = fmaxf(rmax, v);
            }
          rmax = fmaxf(rmax, __shfl_xor_sync(0xffffffffu, rmax, 1));
          rmax = fmaxf(rmax, __shfl_xor_sync(0xffffffffu, rmax, 2));
          if (row >= N) rmax = 0.f;   // padding row: every logit -inf -> E = 0
          float sum = 0.f;
#pragma unroll
          for (int nt = 0; nt < 4; nt++)
#pragma unroll
            for (int u = 0; u < 2; u++) {
              const float ev = fast_ex2(lg[nt][u] - rmax);
              e[mt][nt][2 * h + u] = ev;
              sum += ev;
            }
          sum += __shfl_xor_sync(0xffffffffu, sum, 1);
          sum += __shfl_xor_sync(0xffffffffu, sum, 2);
          const float rs = row < N ? fast_rcp(sum) : 0.f;   // sum >= 1 (the row maximum's term)
#pragma unroll
          for (int nt = 0; nt < 4; nt++)
#pragma unroll
            for (int u = 0; u < 2; u++) e[mt][nt][2 * h + u] *= rs;
        }
      // P' = A X': A fragments from e (k-step kk = j in [16 kk, 16 kk + 16)), B = X' by
      // ldmatrix.trans of the [j][t] rows
      float pacc[2][KT][4];   // [m-tile (rows n)][t-tile][4]
#pragma unroll
      for (int mt = 0; mt < 2; mt++)
#pragma unroll
        for (int tt = 0; tt < KT; tt++)
#pragma unroll
          for (int r = 0; r < 4; r++) pacc[mt][tt][r] = 0.f;
#pragma unroll
      for (int kk = 0; kk < 2; kk++) {
        uint32_t ah[2][4], al[2][4];
#pragma unroll
        for (int mt = 0; mt < 2; mt++) {
          split_pair(e[mt][2 * kk][0], e[mt][2 * kk][1], ah[mt][0], al[mt][0]);
          split_pair(e[mt][2 * kk][2], e[mt][2 * kk][3], ah[mt][1], al[mt][1]);
          split_pair(e[mt][2 * kk + 1][0], e[mt][2 * kk + 1][1], ah[mt][2], al[mt][2]);
          split_pair(e[mt][2 * kk + 1][2], e[mt][2 * kk + 1][3], ah[mt][3], al[mt][3]);
        }
#pragma unroll
        for (int tt = 0; tt < KT; tt++) {
          uint32_t bh0, bh1, bl0, bl1;
          const unsigned char* p = Xh + (16 * kk + (lane & 15)) * PB + 16 * tt;
          ldsm_x2_t(bh0, bh1, p);
          ldsm_x2_t(bl0, bl1, p + K::TILE);
#pragma unroll
          for (int mt = 0; mt < 2; mt++) mma3(pacc[mt][tt], ah[mt], al[mt], bh0, bh1, bl0, bl1);
        }
      }
      // ---------------- gradient: G = dY' P'^T (B fragments from P's accumulators: row n of
      // P' is column n of the B tile), one m-tile of dW at a time
#pragma unroll
      for (int mt = 0; mt < 2; mt++) {
        float gtmp[4][4];
#pragma unroll
        for (int nt = 0; nt < 4; nt++)
#pragma unroll
          for (int r = 0; r < 4; r++) gtmp[nt][r] = 0.f;
#pragma unroll
        for (int kk = 0; kk < KT / 2; kk++) {   // k16 over t-tiles 2 kk, 2 kk + 1
          uint32_t ah[4], al[4];
          const unsigned char* p = Yh + (16 * mt + (lane & 15)) * PB + 2 * (16 * kk + 8 * (lane >> 4));
          ldsm_x4(ah, p);
          ldsm_x4(al, p + K::TILE);
#pragma unroll
          for (int nt = 0; nt < 4; nt++) {   // n = 8 nt + g: row g + 8 (nt & 1) of P's m-tile nt / 2
            const int pm = nt >> 1, ph = nt & 1;
            uint32_t bh0, bl0, bh1, bl1;
            split_pair(pacc[pm][2 * kk][2 * ph], pacc[pm][2 * kk][2 * ph + 1], bh0, bl0);
            split_pair(pacc[pm][2 * kk + 1][2 * ph], pacc[pm][2 * kk + 1][2 * ph + 1], bh1, bl1);
            mma3(gtmp[nt], ah, al, bh0, bh1, bl0, bl1);
          }
        }
        if constexpr (KT & 1) {   // k8 tail over t-tile KT - 1
          uint32_t ah0, ah1, al0, al1;
          const unsigned char* p = Yh + (16 * mt + (lane & 15)) * PB + 2 * (S - 8);
          ldsm_x2(ah0, ah1, p);
          ldsm_x2(al0, al1, p + K::TILE);
#pragma unroll
          for (int nt = 0; nt < 4; nt++) {
            const int pm = nt >> 1, ph = nt & 1;
            uint32_t bh, bl;
            split_pair(pacc[pm][KT - 1][2 * ph], pacc[pm][KT - 1][2 * ph + 1], bh, bl);
            mma3k8(gtmp[nt], ah0, ah1, al0, al1, bh, bl);
          }
        }
#pragma unroll
        for (int nt = 0; nt < 4; nt++)
#pragma unroll
          for (int r = 0; r < 4; r++) acc[br][mt][nt][r] = fmaf(gtmp[nt][r], gsc, acc[br][mt][nt][r]);
      }
    }
  }

  // fixed-order reduction over the warps into this CTA's partial [dW_s | dW_t | db]
  __syncthreads();
  float* red = reinterpret_cast<float*>(smem + (size_t)warp * per_warp);   // [2][32][32]
#pragma unroll
  for (int br = 0; br < 2; br++)
#pragma unroll
    for (int mt = 0; mt < 2; mt++)
#pragma unroll
      for (int nt = 0; nt < 4; nt++)
#pragma unroll
        for (int r = 0; r < 4; r++) {
          const int m = 16 * mt + g + 8 * (r >> 1), n = 8 * nt + 2 * q + (r & 1);
          red[(br * 32 + m) * 32 + n] = acc[br][mt][nt][r];
        }
  __syncthreads();
  const int MN = M * N, E = 2 * MN + H;
  float* out = part + ((int64_t)c * gridDim.x + blockIdx.x) * E;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    float v = 0.f;
    if (e < 2 * MN) {
      const int br = e / MN, mn = e - br * MN, m = mn / N, n = mn - m * N;
      for (int w = 0; w < kBmWarps; w++)
        v += reinterpret_cast<const float*>(smem + (size_t)w * per_warp)[(br * 32 + m) * 32 + n];
    } else {
      const int hh = e - 2 * MN;
      for (int w = 0; w < kBmWarps; w++)
        v += reinterpret_cast<const float*>(smem + (size_t)w * per_warp + K::OFF_DB)[hh];
    }
    out[e] = v;
  }
}

bool bwd_head_mma_shape(const FwdArgs& a) {
  return a.N >= 1 && a.N <= 32 && a.M <= 32 && (a.S == 8 || a.S == 16 || a.S == 24 || a.S == 32) &&
         !a.detrend && !a.revin && !a.comp && a.ma_k == 0;
}

static int bm_per_warp(int S, int H) {
  const int pb = ((S / 8) & 1) ? 2 * S : 2 * S + 16;
  const int tiles = 6 * 32 * pb;
  const int red = 2 * 32 * 32 * 4;   // the final reduction reuses the tile region
  return ((tiles > red ? tiles : red) + 4 * H + 15) & ~15;
}

bool plan_bwd_head_mma(const FwdArgs& a, int max_smem_optin, BwdPlan* p) {
  if (!bwd_head_mma_shape(a)) return false;
  const int pw = bm_per_warp(a.S, a.H);
  const size_t smem = (size_t)kBmWarps * pw;
  if (smem > (size_t)max_smem_optin) return false;
  p->mma_mode = true;
  p->long_mode = false;
  p->warps = kBmWarps;
  p->smem_bytes = smem;
  p->ly.per_warp = pw;
  p->ly.wins_per_cta = 256;   // 32 series per warp
  p->nblk = (int)((a.B + p->ly.wins_per_cta - 1) / p->ly.wins_per_cta);
  p->elems = 2 * a.M * a.N + a.H;
  return true;
}

template <int S>
static cudaError_t launch_bm_t(const FwdArgs& a, const BwdPlan& p, const float* dy, float* part,
                               cudaStream_t st) {
  auto k = prnet_bwd_head_mma_kernel<S>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)p.nblk, (unsigned)a.C);
  k<<<grid, 32 * kBmWarps, p.smem_bytes, st>>>(a, dy, part, p.ly.wins_per_cta, p.ly.per_warp);
  return cudaGetLastError();
}

cudaError_t launch_bwd_head_mma(const FwdArgs& a, const BwdPlan& p, const float* dy, float* part,
                                cudaStream_t st) {
  switch (a.S) {
    case 8: return launch_bm_t<8>(a, p, dy, part, st);
    case 16: return launch_bm_t<16>(a, p, dy, part, st);
    case 24: return launch_bm_t<24>(a, p, dy, part, st);
    default: return launch_bm_t<32>(a, p, dy, part, st);
  }
}

}  // namespace prnet
