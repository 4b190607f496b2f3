// fwd_tcp.cu -- fused PRNet pattern-attention forward, "tc_pipe" variant (S = 24, N <= 32,
// M <= 32): the quad decomposition of tc_quad, re-scheduled so that no warp ever waits for
// a tensor-core round trip it could overlap.
//
// Same reading (SURVEY §8(c) Definition steps 1-11) and split-fp16 3-product
// arithmetic as every other variant.  Per CTA 4 groups x 4 warps; a group
// takes a QUAD of 4 consecutive windows of one channel per round, warp s <-> series s <->
// TMEM lanes 32s..32s+31, lane i <-> segment i.  Per round r a warp runs
//
//   1  a1+a2  series r from its TMA staging row (next series prefetched), descriptors,
//             Z' = z / sqrt(nu2 + eps) and X' = x sx as fp16 hi/lo rows (per-warp tiles;
//             X' double-buffered: the head of round r-1 reads the other buffer)
//   2  a3     seasonal Gram rho = Z' Z'^T on per-warp mma.sync (m16n8k16 + m16n8k8, split
//             fp16): 48 HMMA, no block-diagonal waste, operands in registers (ldmatrix; the
//             B fragments of a Gram ARE the A fragments), the accumulator tiles written to
//             TMEM with tcgen05.st.16x256b (the mma accumulator layout) -> read back
//             lane-per-row with tcgen05.ld.32x32b: TMEM is the transposition engine
//   3  a7+a8  head of quad r-1: wait for its fold (issued at the end of round r-1, so the
//             tensor core had all of steps 1-2 to finish it), Q'^T from TMEM in the 16x256b
//             layout straight into mma.sync A fragments (split + movmatrix), Y' = Q' X' on
//             36 HMMA, streaming stores
//   4  a4+a5  trend and seasonal softmaxes lane-per-row, the transposed attention
//             (symmetric logits, exchanged normalisers; as tc_quad) into TMEM (tcgen05.st)
//   5  a6     arrive on the group's counter (acquire-release atomic); the LAST of the 4
//             warps to arrive issues the fold Q'^T = [A_s^T | A_t^T] W'^T on tcgen05
//             (A from TMEM, the channel head W' from shared memory) and commits it to the
//             group's mbarrier.  No named barriers, no warp blocks on an MMA it just issued.
//
// TMEM (512 columns, 128 per group): [0,32) Gram rows, [32,96) A^T (hi_s | hi_t | lo_s |
// lo_t, fp16 pairs), [96,128) fold accumulator Q'^T.
// Shared memory per warp: TMA staging 3104 B, Z' hi/lo rows (48-byte pitch: conflict-free
// ldmatrix), 2 X' tiles (core-matrix layout for ldmatrix.trans), column vectors; per CTA
// the channel's W' (K-major, pack_tc_head) and bias rows.  One CTA (16 warps) per SM.
//
// Numerical domain as tc_quad: tau_s >= 1/80 (the seasonal shift 1 >= rho_ij keeps the
// largest term of a row >= 2^-ks).
#include <cuda_fp16.h>

#include <cmath>

#include "tc_common.cuh"

namespace prnet {
using namespace tcq;

namespace {

#ifndef PRNET_TCP_SLEEP_NS
#define PRNET_TCP_SLEEP_NS 20000u   // fold-wait suspend hint (ns)
#endif
constexpr int kPGroups = 4;
constexpr int kPWarps = 4 * kPGroups;
// (t - 11.5, t + 1 - 11.5) pairs: the centred positions t~ of Def 3 for S = 24
__constant__ float2 c_tt24[12] = {{-11.5f, -10.5f}, {-9.5f, -8.5f}, {-7.5f, -6.5f}, {-5.5f, -4.5f},
                                  {-3.5f, -2.5f},   {-1.5f, -0.5f}, {0.5f, 1.5f},   {2.5f, 3.5f},
                                  {4.5f, 5.5f},     {6.5f, 7.5f},   {8.5f, 9.5f},   {10.5f, 11.5f}};
constexpr int kPStage = 3104;   // N S fp32 + the sliding mode's alignment slack
constexpr int kPZ = 32 * 48;    // Z' hi (or lo): 32 rows x 24 fp16, 48-byte pitch
constexpr int kPX = 3072;       // one X' tile: 3 t-octets x (hi 512 B | lo 512 B)
constexpr int kPCol = 160 * 4;  // column vectors [5][32] fp32
constexpr int kPWarp = kPStage + 2 * kPZ + 2 * kPX + kPCol;
constexpr int kPOffW = kPWarps * kPWarp;
constexpr int kPBiasRow = 24;   // conflict-free 8-byte epilogue reads (lanes (g, c) -> 24 g + 2 c)
constexpr int kPOffBias = kPOffW + 8192;
constexpr int kPOffBar = kPOffBias + 32 * kPBiasRow * 4;   // 4 fold + 16 TMA mbarriers
constexpr int kPOffCnt = kPOffBar + 8 * (kPGroups + kPWarps);
constexpr int kPOffTmem = kPOffCnt + 4 * kPGroups;
constexpr int kPSmem = kPOffTmem + 16;
static_assert(kPWarp % 16 == 0 && kPStage % 16 == 0, "16-byte aligned tiles");
static_assert(kPSmem <= 227 * 1024, "shared memory");

constexpr uint32_t kIdFold = idesc_f16(128, 32, false, false);

// 8 consecutive fp32 -> 16-byte fp16 hi and lo rows (v = hi + lo)
__device__ __forceinline__ void split8(const float* v, uint4& hi, uint4& lo) {
  uint32_t* h = reinterpret_cast<uint32_t*>(&hi);
  uint32_t* l = reinterpret_cast<uint32_t*>(&lo);
#pragma unroll
  for (int u = 0; u < 4; u++) split2(make_float2(v[2 * u], v[2 * u + 1]), h[u], l[u]);
}
__device__ __forceinline__ void sts128(unsigned char* p, uint4 v) {
  *reinterpret_cast<uint4*>(p) = v;
}

}  // namespace

// NC > 0: compile-time segment count (30: every L = 720, S = 24 config), no column masks;
// NC = 0: runtime N <= 32 with masks.  WIDE: detrended seasonal metric / instance
// normalisation compiled in.  DUMP: the attention rows are also written to a_s_dbg / a_t_dbg
// (prnet_debug_attention), from the same registers the TMEM store takes.
template <int NC, bool WIDE, bool DUMP>
__global__ void __launch_bounds__(512, 1) prnet_fwd_tcp_kernel(FwdArgs a, int ctas_per_channel) {
  const bool detrend = WIDE && a.detrend, revin = WIDE && a.revin;
  static_assert(NC % 2 == 0 && NC <= 32, "NC");
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int S = 24;
  constexpr int NJ = NC > 0 ? NC : 32;   // columns per row (lane-per-row)
  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);
  const int grp = warp >> 2, s = warp & 3;
  const int c = blockIdx.y;
  const int cw = a.head_per_channel ? c : 0;
  const int N = NC > 0 ? NC : a.N;
  const int M = a.M, H = a.H, C = a.C;
  const int i = lane;
  const bool valid = i < N;

  unsigned char* wb = smem + warp * kPWarp;
  float* xstage = reinterpret_cast<float*>(wb);
  unsigned char* zh = wb + kPStage;
  unsigned char* zl = zh + kPZ;
  unsigned char* xt0 = zl + kPZ;
  // column vectors: [0] mu~, [1] kappa~, [2] 1/l_t, [3] 1/l_s, [4] seasonal mask (NC = 0)
  float* colv = reinterpret_cast<float*>(xt0 + 2 * kPX);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kPOffBar);
  uint64_t* fbar = bars + grp;                 // the group's fold completion
  uint64_t* xbar = bars + kPGroups + warp;     // this warp's TMA load
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + kPOffCnt) + grp;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kPOffTmem);
  const float* bS = reinterpret_cast<const float*>(smem + kPOffBias);

  // ---------------- prologue: channel head W' and bias, barriers, counters, TMEM.  The
  // operand tiles need no zero fill: every row an active series reads is written each round.
  {
    const uint4* src = a.wpack_tc + (int64_t)cw * (8192 / 16);
    uint4* dst = reinterpret_cast<uint4*>(smem + kPOffW);
    for (int k = threadIdx.x; k < 8192 / 16; k += blockDim.x) dst[k] = __ldg(src + k);
    const float* gb = a.bias + (int64_t)cw * H;
    float* bw = reinterpret_cast<float*>(smem + kPOffBias);
    for (int k = threadIdx.x; k < 32 * kPBiasRow; k += blockDim.x) {
      const int h = (k / kPBiasRow) * 24 + k % kPBiasRow;
      bw[k] = h < H ? __ldg(gb + h) : 0.f;
    }
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < kPGroups + kPWarps; k++) mbar_init(bars + k, 1);
    for (int k = 0; k < kPGroups; k++) reinterpret_cast<uint32_t*>(smem + kPOffCnt)[k] = 0u;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem0 = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const uint32_t tcol = tmem0 + 128u * (uint32_t)grp;   // the group's 128 columns
  const uint32_t tlane = (uint32_t)(32 * s) << 16;        // this warp's 32 lanes
  const uint32_t tG = tcol + tlane, tA = tcol + 32u + tlane, tF = tcol + 96u + tlane;
  const uint32_t w_s = smem_u32(smem + kPOffW);
  const float inv_sw = __ldg(a.wpack_inv_sw + cw);
  const bool full_rows = H == 24 * M && (H & 1) == 0;   // the output rows tile H exactly

  // windows of channel c: CTA k of the channel takes [B k / K, B (k+1) / K), split into
  // near-equal runs of whole quads over the groups
  const int64_t cb0 = a.B * blockIdx.x / ctas_per_channel;
  const int64_t cb1 = a.B * (blockIdx.x + 1) / ctas_per_channel;
  const int64_t quads = (cb1 - cb0 + 3) / 4;
  const int64_t g0 = cb0 + 4 * (quads * grp / kPGroups);
  const int64_t g1 = min(cb0 + 4 * (quads * (grp + 1) / kPGroups), cb1);
  const int rounds = g1 > g0 ? (int)((g1 - g0 + 3) / 4) : 0;
  const int NS = N * S;
  const bool bulk = a.x_vec;
  const int64_t win0 = g0 + s;
  const float* xnext = a.x + win0 * a.xsb + c * a.xsc + a.r;
  float* ycur = a.y + (win0 * C + c) * H;
  const int64_t xstep = 4 * a.xsb, ystep = 4 * (int64_t)C * H;
  // sliding windows (prnet_forward_sliding, window starts not 16-byte aligned): one 1-D bulk
  // copy of the aligned superset [floor4(start), ceil4(start + NS)) when it stays inside the
  // series buffer; the window then starts o = start mod 4 floats into the staging row
  const bool slide = !bulk && a.x_end != nullptr;
  auto slide_o = [&](const float* xg) { return (int)(((uintptr_t)xg >> 2) & 3u); };
  auto slide_bytes = [&](const float* xg) { return (uint32_t)((slide_o(xg) + NS + 3) & ~3) * 4u; };
  auto slide_bulk = [&](const float* xg) {
    return slide && ((uintptr_t)xg & ~(uintptr_t)15) + slide_bytes(xg) <= (uintptr_t)a.x_end;
  };
  auto issue_load = [&](const float* xg) {
    if (bulk) {
      if (lane == 0) bulk_load(xstage, xg, (uint32_t)NS * 4u, xbar);
    } else if (slide_bulk(xg)) {
      if (lane == 0)
        bulk_load(xstage, reinterpret_cast<const float*>((uintptr_t)xg & ~(uintptr_t)15),
                  slide_bytes(xg), xbar);
    } else {
      const int o = slide ? slide_o(xg) : 0;
      for (int k = lane; k < NS; k += 32) cp_async4(xstage + o + k, xg + k);
      cp_async_commit();
    }
  };

  // the previous round's series, whose head runs in this round (step 3)
  bool pact = false;
  float psx = 1.f, psr = 1.f, pmr = 0.f;
  float* pycur = ycur;
  uint32_t xph = 0;
  if (rounds > 0 && win0 < g1) issue_load(xnext);
  for (int rd = 0; rd <= rounds; rd++) {
    const int64_t b = g0 + 4 * rd + s;
    const bool active = rd < rounds && b < g1;
    float sx = 1.f, sr = 1.f, mr = 0.f, mi = 0.f, ki = 0.f;
    unsigned char* xt = xt0 + (rd & 1) * kPX;

    if (active) {
      // ---------------- 1  a1+a2: segment row i (Def 2) from the TMA staging, descriptors
      // (Def 4-5) from d = x - x0 (a constant segment gives exact zeros), Z' and X' rows
      float xv[24];
      if (bulk || slide_bulk(xnext)) {
        mbar_wait_bounded(xbar, xph);
        xph ^= 1u;
      } else {
        cp_async_wait_all();
      }
      __syncwarp();
      float dv[24];
      {
        const int o = slide ? slide_o(xnext) : 0;   // warp-uniform
        const float4* xr = reinterpret_cast<const float4*>(xstage + (valid ? i : N - 1) * 24);
        if (o == 0) {
          // rows are 96 B apart, so lanes i and i + 4 of a quarter-warp hit the same banks:
          // lanes with (i / 4) odd read the float4s in rotated order (q + 1) mod 6 and the
          // registers are rotated back with selects (no bank conflicts)
          const bool rot = (i >> 2) & 1;
          float4 v[6];
#pragma unroll
          for (int q = 0; q < 6; q++) v[q] = xr[rot ? (q + 1) % 6 : q];
#pragma unroll
          for (int q = 0; q < 6; q++) {
            const float4 u = rot ? v[(q + 5) % 6] : v[q];
            xv[4 * q] = u.x;
            xv[4 * q + 1] = u.y;
            xv[4 * q + 2] = u.z;
            xv[4 * q + 3] = u.w;
          }
        } else {
          // the row starts o floats past an aligned address: 7 aligned loads, static shift
          float w[28];
#pragma unroll
          for (int q = 0; q < 7; q++) {
            const float4 v = xr[q];
            w[4 * q] = v.x;
            w[4 * q + 1] = v.y;
            w[4 * q + 2] = v.z;
            w[4 * q + 3] = v.w;
          }
          if (o == 1) {
#pragma unroll
            for (int t = 0; t < 24; t++) xv[t] = w[t + 1];
          } else if (o == 2) {
#pragma unroll
            for (int t = 0; t < 24; t++) xv[t] = w[t + 2];
          } else {
#pragma unroll
            for (int t = 0; t < 24; t++) xv[t] = w[t + 3];
          }
        }
      }
      __syncwarp();
      // the staging row is in registers: fetch this warp's next series now
      xnext += xstep;
      if (b + 4 < g1) issue_load(xnext);
      const float x0 = xv[0];
      float2 s1 = f2(0.f), s3 = f2(0.f);
#pragma unroll
      for (int t = 0; t < 24; t += 2) {
        const float2 d = add2(make_float2(xv[t], xv[t + 1]), f2(-x0));
        dv[t] = d.x;
        dv[t + 1] = d.y;
        s1 = add2(s1, d);
        s3 = fma2(c_tt24[t / 2], d, s3);
      }
      const float m1 = (s1.x + s1.y) * (1.f / 24.f);
      const float mu = x0 + m1;
      const float s3s = s3.x + s3.y;
      const float kap = s3s * a.inv_v;
      float2 q2 = f2(0.f);
      const float2 nm1 = f2(-m1);
      if (!detrend) {
#pragma unroll
        for (int t = 0; t < 24; t += 2) {
          const float2 z = add2(make_float2(dv[t], dv[t + 1]), nm1);
          dv[t] = z.x;
          dv[t + 1] = z.y;
          q2 = fma2(z, z, q2);
        }
      } else {
        // metric_variant bit 1: the seasonal metric sees the residual
        // e = z - kappa t~ about the segment's least-squares line
        const float2 nk2 = f2(-kap);
#pragma unroll
        for (int t = 0; t < 24; t += 2) {
          const float2 e = fma2(nk2, c_tt24[t / 2], add2(make_float2(dv[t], dv[t + 1]), nm1));
          dv[t] = e.x;
          dv[t + 1] = e.y;
          q2 = fma2(e, e, q2);
        }
      }
      const float nu2s = q2.x + q2.y;                        // |z|^2, or |e|^2 (detrended)
      // Def 4: nu2 = |z|^2 = |e|^2 + kappa^2 V (e orthogonal to t~) for Def 5
      const float nu2 = detrend ? fmaf(s3s, kap, nu2s) : nu2s;
      // Z' = (e or z) rr / sqrt(nu2 rr^2 + eps_s) and X' = (x - mu_r) rr sx as split-fp16 rows
      // of the Gram / head operand tiles.  Plain path (rr = 1, mu_r = 0): written before the
      // sigma^2 shuffle tree, off its dependency chain; instance_norm: after it.
      auto write_operands = [&](float mu_r, float rr) {
        const float zsc = rr * rsqrtf(nu2s * rr * rr + kEpsSeasonal);
        // |xhat_t| <= (|mu - mu_r| + |kappa| 11.5 [detrended] + |e or z|) rr: an exact
        // power-of-two scale for X' from it
        const float bnd =
            (fabsf(mu - mu_r) + (detrend ? 11.5f * fabsf(kap) : 0.f) + sqrtf(nu2s)) * rr;
        sx = pow2_scale(warp_max_nonneg(valid ? bnd : 0.f));
        const float2 zs2 = f2(valid ? zsc : 0.f), xs2 = f2(valid ? rr * sx : 0.f);
        const float2 xo2 = f2(valid ? -mu_r * rr * sx : 0.f);
#pragma unroll
        for (int t = 0; t < 24; t += 2) {
          const float2 zz = mul2(make_float2(dv[t], dv[t + 1]), zs2);
          const float2 xx = fma2(make_float2(xv[t], xv[t + 1]), xs2, xo2);
          dv[t] = zz.x;
          dv[t + 1] = zz.y;
          xv[t] = xx.x;
          xv[t + 1] = xx.y;
        }
        unsigned char* zr = zh + i * 48;
        unsigned char* xr = xt + (i >> 3) * 128 + (i & 7) * 16;
#pragma unroll
        for (int q = 0; q < 3; q++) {
          uint4 h, l;
          split8(dv + 8 * q, h, l);
          sts128(zr + q * 16, h);
          sts128(zr + kPZ + q * 16, l);
          split8(xv + 8 * q, h, l);
          sts128(xr + q * 1024, h);
          sts128(xr + q * 1024 + 512, l);
        }
      };
      if (!revin) write_operands(0.f, 1.f);
      // Def 5: sigma^2 = (1/(N S)) sum_n [nu2_n + S (mu_n - mubar)^2], both sums in one
      // shuffle tree about the reference m0 = mu_0 (exact regrouping)
      const float m0 = __shfl_sync(0xffffffffu, mu, 0);
      const float dd = valid ? mu - m0 : 0.f;
      float2 acc = make_float2(dd, valid ? fmaf(24.f * dd, dd, nu2) : 0.f);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        acc = add2(acc, make_float2(__shfl_xor_sync(0xffffffffu, acc.x, o),
                                    __shfl_xor_sync(0xffffffffu, acc.y, o)));
      const float var = fmaf(-24.f * acc.x, acc.x * a.inv_n, acc.y) * a.inv_ns;
      // instance normalisation: every descriptor of xhat is an affine
      // image of the descriptor of x, so only scalars change.  Off: mu_r = 0, rr = sr = 1.
      float mu_r = 0.f, rr = 1.f;
      if (revin) {
        mu_r = fmaf(acc.x, a.inv_n, m0);
        rr = rsqrtf(var + kEpsRevin);
        sr = (var + kEpsRevin) * rr;
        mr = mu_r;
        write_operands(mu_r, rr);
      }
      const float inv_var = 1.0f / fmaf(var * rr, rr, kEpsTrend);
      // trend (Def 7-8): exponent -(mu~_i - mu~_j)^2 - (k~_i - k~_j)^2, mu~ = muhat sqrt(kt/var'),
      // k~ = kappahat sqrt(vtrend kt/var')
      mi = (mu - mu_r) * rr * sqrtf(inv_var * a.kt);
      ki = kap * rr * sqrtf(a.vtrend * inv_var * a.kt);
      colv[i] = (NC > 0 || valid) ? mi : INFINITY;   // -> exponent -inf past N
      colv[32 + i] = ki;
      if constexpr (NC == 0) colv[128 + i] = valid ? 0.f : -INFINITY;
      __syncwarp();

      // ---------------- 2  a3: Gram rho = Z' Z'^T on mma.sync, 3 split products, fp32
      // accumulators -> TMEM columns [0, 32) of this warp's lanes (16x256b = mma layout)
      {
        uint32_t ah[2][4], al[2][4], ah8[4], al8[4];
        {
          const int l8 = lane & 7, q = lane >> 3;
#pragma unroll
          for (int mt = 0; mt < 2; mt++) {
            const unsigned char* p = zh + (16 * mt + (q & 1) * 8 + l8) * 48 + (q >> 1) * 16;
            ldsm_x4(ah[mt], p);
            ldsm_x4(al[mt], p + kPZ);
          }
          const unsigned char* p8 = zh + lane * 48 + 32;
          ldsm_x4(ah8, p8);
          ldsm_x4(al8, p8 + kPZ);
        }
        // issue order: product-major, 8 independent accumulators between dependent MMAs
        // (hi-lo cross terms first, hi-hi last)
        float g[2][16];
#pragma unroll
        for (int mt = 0; mt < 2; mt++)
#pragma unroll
          for (int e = 0; e < 16; e++) g[mt][e] = 0.f;
#define PRNET_GRAM_PASS(A16, A8, B16, B8)                                                  \
  _Pragma("unroll") for (int mt = 0; mt < 2; mt++)                                         \
  _Pragma("unroll") for (int nt = 0; nt < 4; nt++) {                                       \
    float(&acc4)[4] = *reinterpret_cast<float(*)[4]>(&g[mt][4 * nt]);                      \
    mma16816_nv(acc4, A16[mt], B16[nt >> 1][nt & 1], B16[nt >> 1][2 + (nt & 1)]);          \
    mma1688_nv(acc4, A8[2 * mt], A8[2 * mt + 1], B8[nt]);                                   \
  }
        // B fragments of the Gram = A fragments of rows 8 nt .. 8 nt + 7
        PRNET_GRAM_PASS(al, al8, ah, ah8)
        PRNET_GRAM_PASS(ah, ah8, al, al8)
        PRNET_GRAM_PASS(ah, ah8, ah, ah8)
#undef PRNET_GRAM_PASS
        tst16_x4(tG, g[0]);
        tst16_x4(tG + (16u << 16), g[1]);
      }
    }

    // ---------------- 4s  a5 seasonal softmax from the Gram row (lane j -> column j of A_s,
    // E_ij = 2^((rho_ij - 1) ks)); its A^T half is parked in the Gram columns until the
    // fold of the previous quad has released the A^T columns (step 5)
    if (active) {
      const int64_t series = b * C + c;   // debug_attention row block
      uint32_t sh[16], sl[16];
      {
        uint32_t gr[32];
        tst_wait();   // (the Gram tiles of step 2 were stored by this warp)
        tld_x32(tG, gr);
        tld_wait();
        float e[32];
        const float2 ks2 = f2(a.ks), nks2 = f2(-a.ks);
        const float4* cx4 = reinterpret_cast<const float4*>(colv + 128);
        float2 sum2 = f2(0.f);
#pragma unroll
        for (int j = 0; j < NJ; j += 2) {
          float2 arg = fma2(make_float2(__uint_as_float(gr[j]), __uint_as_float(gr[j + 1])), ks2,
                            nks2);
          if constexpr (NC == 0) {
            const float4 mk = cx4[j >> 2];
            arg = add2(arg, (j & 2) ? make_float2(mk.z, mk.w) : make_float2(mk.x, mk.y));
          }
          e[j] = fast_ex2(arg.x);
          e[j + 1] = fast_ex2(arg.y);
          sum2 = add2(sum2, make_float2(e[j], e[j + 1]));
        }
        colv[96 + i] = valid ? fast_rcp(sum2.x + sum2.y) : 0.f;
        __syncwarp();
        const float4* cr4 = reinterpret_cast<const float4*>(colv + 96);
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const float4 r = cr4[q];
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int j = 4 * q + 2 * h;
            if (j >= NJ) {
              sh[j / 2] = 0u;
              sl[j / 2] = 0u;
              continue;
            }
            const float2 v = mul2(make_float2(e[j], e[j + 1]), h ? make_float2(r.z, r.w) : make_float2(r.x, r.y));
            if constexpr (DUMP) {
              if (valid) {
                float* d = a.a_s_dbg + series * N * N + lane;
                if (j < N) d[(int64_t)j * N] = v.x;
                if (j + 1 < N) d[(int64_t)(j + 1) * N] = v.y;
              }
            }
            split2(v, sh[j / 2], sl[j / 2]);
          }
        }
      }
      tst_x16(tG, sh);
      tst_x16(tG + 16u, sl);
    }

    // ---------------- 3  a7 + a8: head of the previous quad (its fold ran during steps 1-2)
    if (rd > 0) {
      mbar_wait_sleep(fbar, (uint32_t)(rd - 1) & 1u, PRNET_TCP_SLEEP_NS);
      tc_fence_after();
    }
    if (pact) {
      // Q'^T straight into the head's A fragments: 16x256b loads give 8x8 blocks of Q'^T
      // (rows j, columns m) in the mma accumulator layout; split to fp16 hi/lo and
      // transposed in registers (movmatrix): block (j-half h, j-octet v, m-octet k) is
      // A-fragment register (k & 1) + 2v of tile (m-tile k / 2, k-tile h)
      uint32_t qah[2][2][4], qal[2][2][4];   // [mt][kt][reg]
      {
        uint32_t r0[16], r1[16];
        tld16_x4(tF, r0);
        tld16_x4(tF + (16u << 16), r1);
        tld_wait();
#pragma unroll
        for (int h = 0; h < 2; h++)
#pragma unroll
          for (int v = 0; v < 2; v++)
#pragma unroll
            for (int k = 0; k < 4; k++) {
              const uint32_t* r = h ? r1 : r0;
              uint32_t hi, lo;
              split2(make_float2(__uint_as_float(r[4 * k + 2 * v]),
                                 __uint_as_float(r[4 * k + 2 * v + 1])),
                     hi, lo);
              qah[k >> 1][h][(k & 1) + 2 * v] = movm_t(hi);
              qal[k >> 1][h][(k & 1) + 2 * v] = movm_t(lo);
            }
      }
      // Y' = Q' X' with m16n8k16 split-fp16 MMAs, X' B fragments by ldmatrix.trans
      const unsigned char* xs = xt0 + ((rd - 1) & 1) * kPX;
      const int l8 = lane & 7, g4 = lane >> 3;
      float acc[2][3][4];
#pragma unroll
      for (int mt = 0; mt < 2; mt++)
#pragma unroll
        for (int nt = 0; nt < 3; nt++)
#pragma unroll
          for (int e = 0; e < 4; e++) acc[mt][nt][e] = 0.f;
#pragma unroll
      for (int kt = 0; kt < 2; kt++) {
        // B = X'[j][t]: (j-block 2kt + (g4 & 1), t-block nt + (g4 >> 1)) for the x4 pair
        uint32_t xh[3][2], xl[3][2];
        {
          uint32_t r[4];
          const unsigned char* p = xs + (g4 >> 1) * 1024 + (2 * kt + (g4 & 1)) * 128 + l8 * 16;
          ldsm_x4_t(r, p);
          xh[0][0] = r[0]; xh[0][1] = r[1]; xh[1][0] = r[2]; xh[1][1] = r[3];
          ldsm_x4_t(r, p + 512);
          xl[0][0] = r[0]; xl[0][1] = r[1]; xl[1][0] = r[2]; xl[1][1] = r[3];
          const unsigned char* p2 = xs + 2 * 1024 + (2 * kt + (g4 & 1)) * 128 + l8 * 16;
          ldsm_x2_t(xh[2][0], xh[2][1], p2);
          ldsm_x2_t(xl[2][0], xl[2][1], p2 + 512);
        }
        // product-major: 6 independent accumulators between dependent MMAs
#pragma unroll
        for (int mt = 0; mt < 2; mt++)
#pragma unroll
          for (int nt = 0; nt < 3; nt++) mma16816_nv(acc[mt][nt], qal[mt][kt], xh[nt][0], xh[nt][1]);
#pragma unroll
        for (int mt = 0; mt < 2; mt++)
#pragma unroll
          for (int nt = 0; nt < 3; nt++) mma16816_nv(acc[mt][nt], qah[mt][kt], xl[nt][0], xl[nt][1]);
#pragma unroll
        for (int mt = 0; mt < 2; mt++)
#pragma unroll
          for (int nt = 0; nt < 3; nt++) mma16816_nv(acc[mt][nt], qah[mt][kt], xh[nt][0], xh[nt][1]);
      }
      // a8 store: y = Y' / (sw sx) + b (Def 11), pairs (m, t..t+1)
      const float2 ys2 = f2(inv_sw * psr / psx);
      const float2 sr2 = f2(psr), mr2 = f2(pmr);
      float* yg = pycur + 2 * (lane & 3);
      const float* bq = bS + 2 * (lane & 3);
      if (full_rows) {   // H = 24 M, H even: every (m < M, t) pair is stored, no tail
#pragma unroll
        for (int mt = 0; mt < 2; mt++)
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int m = 16 * mt + 8 * h + (lane >> 2);
            if (m < M) {
              float* yr = yg + m * 24;
              const float* br = bq + m * kPBiasRow;
#pragma unroll
              for (int nt = 0; nt < 3; nt++) {
                float2 bb = *reinterpret_cast<const float2*>(br + 8 * nt);
                if (revin) bb = fma2(bb, sr2, mr2);   // y = yhat sr + mr
                const float2 o =
                    fma2(make_float2(acc[mt][nt][2 * h], acc[mt][nt][2 * h + 1]), ys2, bb);
                asm volatile("st.global.cs.v2.f32 [%0], {%1,%2};" ::"l"(yr + 8 * nt), "f"(o.x),
                             "f"(o.y)
                             : "memory");
              }
            }
          }
      } else {
#pragma unroll
        for (int mt = 0; mt < 2; mt++)
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int m = 16 * mt + 8 * h + (lane >> 2);
            if (m >= M) continue;
#pragma unroll
            for (int nt = 0; nt < 3; nt++) {
              const int hh = m * 24 + 8 * nt + 2 * (lane & 3);
              float2 bb = *reinterpret_cast<const float2*>(bq + m * kPBiasRow + 8 * nt);
              if (revin) bb = fma2(bb, sr2, mr2);
              const float2 o = fma2(make_float2(acc[mt][nt][2 * h], acc[mt][nt][2 * h + 1]), ys2, bb);
              if (hh < H) yg[m * 24 + 8 * nt] = o.x;
              if (hh + 1 < H) yg[m * 24 + 8 * nt + 1] = o.y;
            }
          }
      }
    }
    if (rd == rounds) break;

    // ---------------- 4t  a4+a5 trend softmax: lane j -> column j of A_t, A_t[i][j] = E_ji / l_i
    // (E symmetric, shift 0 = the row max, attained at j = i); then A^T = [A_s | A_t] hi/lo
    // into TMEM columns [32, 96) (the fold of the previous quad finished reading them: step 3)
    if (active) {
      const int64_t series = b * C + c;
      uint32_t th[16], tl[16];
      {
        float e[32];
        const float2 mi2 = f2(mi), ki2 = f2(ki);
        float2 sum2 = f2(0.f);
        const float4* cm4 = reinterpret_cast<const float4*>(colv);
        const float4* ck4 = reinterpret_cast<const float4*>(colv + 32);
#pragma unroll
        for (int q = 0; q < 8; q++) {
          if (4 * q >= NJ) break;
          const float4 mj = cm4[q], kj = ck4[q];
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int j = 4 * q + 2 * h;
            if (j >= NJ) break;
            const float2 dmj = add2(mi2, h ? make_float2(-mj.z, -mj.w) : make_float2(-mj.x, -mj.y));
            const float2 dkj = add2(ki2, h ? make_float2(-kj.z, -kj.w) : make_float2(-kj.x, -kj.y));
            const float2 ex =
                fma2(make_float2(-dkj.x, -dkj.y), dkj, mul2(make_float2(-dmj.x, -dmj.y), dmj));
            e[j] = fast_ex2(ex.x);
            e[j + 1] = fast_ex2(ex.y);
            sum2 = add2(sum2, make_float2(e[j], e[j + 1]));
          }
        }
        colv[64 + i] = valid ? fast_rcp(sum2.x + sum2.y) : 0.f;
        __syncwarp();
        const float4* cr4 = reinterpret_cast<const float4*>(colv + 64);
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const float4 r = cr4[q];
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int j = 4 * q + 2 * h;
            if (j >= NJ) {
              th[j / 2] = 0u;
              tl[j / 2] = 0u;
              continue;
            }
            const float2 v = mul2(make_float2(e[j], e[j + 1]), h ? make_float2(r.z, r.w) : make_float2(r.x, r.y));
            if constexpr (DUMP) {
              if (valid) {
                float* d = a.a_t_dbg + series * N * N + lane;
                if (j < N) d[(int64_t)j * N] = v.x;
                if (j + 1 < N) d[(int64_t)(j + 1) * N] = v.y;
              }
            }
            split2(v, th[j / 2], tl[j / 2]);
          }
        }
      }
      uint32_t ss[32];   // the parked seasonal half: sh | sl
      tst_wait();
      tld_x32(tG, ss);
      tld_wait();
      tst_x16(tA, *reinterpret_cast<const uint32_t(*)[16]>(ss));
      tst_x16(tA + 16u, th);
      tst_x16(tA + 32u, *reinterpret_cast<const uint32_t(*)[16]>(ss + 16));
      tst_x16(tA + 48u, tl);
      tst_wait();
    }

    // ---------------- 5  a6 fold on tcgen05, issued by the last warp of the group to arrive:
    // Q'^T = [A_s^T | A_t^T] W'^T (Def 9-10 folded), A from TMEM, W' from shared memory
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      const uint32_t old = atom_add_acqrel(cnt, 1u);
      if ((old & 3u) == 3u) {
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < 4; ks++) {
          const uint64_t bh = sdesc(w_s + ks * 256, 128, 2048);
          const uint64_t bl = sdesc(w_s + (8 + 2 * ks) * 128, 128, 2048);
          umma_ts(tcol + 96u, tcol + 32u + 8u * ks, bh, kIdFold, ks > 0);
          umma_ts(tcol + 96u, tcol + 32u + 8u * ks, bl, kIdFold, true);
          umma_ts(tcol + 96u, tcol + 64u + 8u * ks, bh, kIdFold, true);
        }
        umma_commit(fbar);
      }
    }
    __syncwarp();
    pact = active;
    psx = sx;
    psr = sr;
    pmr = mr;
    pycur = ycur;
    ycur += ystep;
  }
  cp_async_wait_all();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem0, 512);
}

bool plan_tcp_kernel(const FwdArgs& a, int max_smem_optin, int sm_count, TcqPlan* p) {
  if (a.S != 24 || a.N < 1 || a.N > 32 || a.M > 32) return false;
  p->smem_bytes = (size_t)kPSmem;
  if (p->smem_bytes > (size_t)max_smem_optin) return false;
  p->wins_per_group = 128;
  // one CTA per SM: a small launch (few channels x few windows) ends in a partial wave.
  // Split each channel into k CTAs, k >= B / (4 x 128), minimising
  //   waves(k) x (windows per CTA + kPrologue)
  // where kPrologue ~ the per-CTA setup (W' and bias loads, TMEM allocation) in windows
  constexpr int64_t kPrologue = 32;
  const int64_t per_cta = (int64_t)kPGroups * p->wins_per_group;
  const int64_t k0 = a.B > 0 ? (a.B + per_cta - 1) / per_cta : 1;
  const int64_t sms = sm_count > 0 ? sm_count : 148;
  int64_t best_k = k0, best = -1;
  for (int64_t k = k0; k <= 4 * k0 && k <= (a.B + 63) / 64 + 1; k++) {
    const int64_t waves = ((int64_t)a.C * k + sms - 1) / sms;
    const int64_t cost = waves * ((a.B + k - 1) / k + kPrologue);
    if (best < 0 || cost < best) best = cost, best_k = k;
  }
  p->ctas_per_channel = (int)best_k;
  return true;
}

template <int NC, bool WIDE, bool DUMP>
static cudaError_t launch_tcp_t(const FwdArgs& a, const TcqPlan& p, cudaStream_t st) {
  auto k = prnet_fwd_tcp_kernel<NC, WIDE, DUMP>;
  cudaError_t e =
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  const int64_t per_cta = (int64_t)kPGroups * p.wins_per_group;
  const int ctas =
      p.ctas_per_channel > 0 ? p.ctas_per_channel : (int)((a.B + per_cta - 1) / per_cta);
  dim3 grid((unsigned)ctas, (unsigned)a.C);
  k<<<grid, 32 * kPWarps, p.smem_bytes, st>>>(a, ctas);
  return cudaGetLastError();
}

cudaError_t launch_tcp_kernel(const FwdArgs& a, const TcqPlan& p, cudaStream_t st) {
  if (a.a_s_dbg != nullptr) return launch_tcp_t<0, true, true>(a, p, st);
  const bool wide = a.detrend || a.revin;
  if (a.N == 30) return wide ? launch_tcp_t<30, true, false>(a, p, st) : launch_tcp_t<30, false, false>(a, p, st);
  return wide ? launch_tcp_t<0, true, false>(a, p, st) : launch_tcp_t<0, false, false>(a, p, st);
}

}  // namespace prnet
