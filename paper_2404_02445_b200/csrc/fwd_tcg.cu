// fwd_tcg.cu -- the tc_quad organisation (fwd_tcq.cu) for segment lengths other than 24:
// S in {12, 16, 32, 48, 64, 96} (compile-time instantiations), N <= 32, M <= 32.
//
// Same reading (SURVEY §8(c) Definition steps 1-11) and split-fp16 3-product
// arithmetic as every other variant.  The work decomposition is tc_quad's:
// a group of 4 warps runs a QUAD of 4 series (consecutive windows of one channel) per round,
// warp s <-> series s <-> TMEM lanes 32s..32s+31, lane i <-> segment i; the seasonal Gram
// of the row-normalised Z' and the fold Q'^T = [A_s^T | A_t^T] W'^T run on tcgen05.mma with
// TMEM accumulators, the softmaxes lane-per-row (symmetric logits: lane j computes row j
// of E, which is column j; only the normalisers 1/l_i are exchanged), the head on per-warp
// mma.sync.  What changes with S:
//
//  * the segment rows are streamed from the staging area in float4 chunks in three passes
//    (sums, centred square sum, operand rows), so no lane holds a whole row in registers
//    (S = 96 would need 192 of them);
//  * staging rows are PITCH bytes apart, PITCH/16 odd (conflict-free quarter-warp float4
//    reads); when 4S/16 is even the series is fetched by one 1-D bulk copy per segment row
//    (lane n issues row n), else by one bulk copy of the whole N S span;
//  * the Gram K is S padded to SP = 16k per product, the three products hh, hl, lh are three
//    runs of SP/16 K-steps over one [hi | lo] row tile (no duplicated chunk);
//  * the head's X' tile of series s lives in warp s's quarter of the Z' tile (its rows
//    32s..32s+31 are one contiguous quarter, 128 SP bytes >= the 1024 ceil(S/8) X' bytes) and
//    is written after the Gram completes: no cross-warp hazard, no extra shared memory;
//  * the head runs in groups of n-tiles (8 t each) to bound the accumulator registers and
//    skips the second m-tile when M <= 16.
//
// Numerical domain: tau_s >= 1/80 (the seasonal shift 1, as tc_quad).
#include <cuda_fp16.h>

#include <cmath>

#include "tc_common.cuh"

namespace prnet {
using namespace tcq;

namespace {

template <int S, bool M64 = false>
struct TcgCfg {
  static_assert(S % 4 == 0 && S >= 8 && S <= 96, "S");
  static constexpr int SP = (S + 15) / 16 * 16;   // Gram K per product (t zero-padded)
  static constexpr int NCT = (S + 7) / 8;         // head n-tiles of 8 t
  static constexpr int NQ = S / 4;                // float4 chunks per segment row
  static constexpr int PITCH = ((S / 4) & 1) ? 4 * S : 4 * S + 16;   // staging row bytes
  static constexpr bool ROWCOPY = PITCH != 4 * S;
  static constexpr int SBO = 32 * SP;             // Z' row-block (8 rows) stride, bytes
  static constexpr int ZQ = 128 * SP;             // one warp's quarter: its 32 Z' rows | X'
  static constexpr int ZT = 4 * ZQ;
  static constexpr int STAGE = 32 * PITCH;        // per warp staging (N <= 32 rows)
  static constexpr int COLV = 160 * 4;            // per warp column vectors [5][32] fp32
  static constexpr int GROUP = ZT + 4 * STAGE + 4 * COLV;
  static constexpr int BR = (NCT & 1) ? 8 * NCT : 8 * NCT + 8;   // bias row stride (floats)
  static constexpr int WB = M64 ? 16384 : 8192;                   // W' tile (32 or 64 m-rows)
  static constexpr int FIXED = WB + 256 + 16 + (M64 ? 64 : 32) * BR * 4;   // W', bars, slot, bias
  static_assert(ZQ >= NCT * 1024, "X' fits the quarter");
  // groups per CTA that fit the 227 KB opt-in shared memory (the launch-bounds thread count)
  static constexpr int MAXG = (232448 - FIXED) / GROUP >= 4 ? 4 : (232448 - FIXED) / GROUP;
  static_assert(MAXG >= 1, "one group fits");
};

constexpr uint32_t kIdGramG = idesc_f16(128, 128, false, false);
constexpr uint32_t kIdFoldG = idesc_f16(128, 32, false, false);
constexpr uint32_t kIdFoldG64 = idesc_f16(128, 64, false, false);
constexpr uint32_t kIdFoldG16 = idesc_f16(128, 16, false, false);   // M <= 16: one head m-tile

__device__ __forceinline__ void sts128(unsigned char* p, uint4 v) {
  *reinterpret_cast<uint4*>(p) = v;
}
__device__ __forceinline__ void bulk_copy_nobar_expect(void* dst, const void* src, uint32_t bytes,
                                                       uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// position t~ = t - (S - 1) / 2 of Def 3 (compile-time for the unrolled chunk loops)
template <int S>
__device__ __forceinline__ constexpr float ttl(int t) {
  return (float)t - 0.5f * (float)(S - 1);
}

}  // namespace

// DUMP (prnet_debug_attention): the attention values each lane hands to the TMEM store are
// also written to a_s_dbg / a_t_dbg from the same registers.
template <int S, bool DUMP, bool M64>
__global__ void __launch_bounds__(128 * TcgCfg<S, M64>::MAXG, 1) prnet_fwd_tcg_kernel(FwdArgs a, int ctas_per_channel) {
  using K = TcgCfg<S, M64>;
  extern __shared__ __align__(1024) unsigned char smem[];
  const int ngroups = blockDim.x >> 7;
  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);
  const int grp = warp >> 2, s = warp & 3;
  const int c = blockIdx.y;
  const int cw = a.head_per_channel ? c : 0;
  const int N = a.N, M = a.M, H = a.H, C = a.C;
  const int i = lane;
  const bool valid = i < N;

  unsigned char* gbase = smem + grp * K::GROUP;
  unsigned char* zt = gbase;                     // Z' tile; quarter s doubles as X' of series s
  unsigned char* xq = zt + s * K::ZQ;            // this warp's quarter
  unsigned char* stage = gbase + K::ZT + s * K::STAGE;
  float* colv = reinterpret_cast<float*>(gbase + K::ZT + 4 * K::STAGE) + s * 160;
  const int offw = ngroups * K::GROUP;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + offw + K::WB);
  uint64_t* mbar = bars + 2 * grp;                 // +0 Gram, +1 fold
  uint64_t* xbar = bars + 8 + warp;                // this warp's load
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + offw + K::WB + 256);
  float* bS = reinterpret_cast<float*>(smem + offw + K::WB + 256 + 16);

  // ---------------- prologue: channel head W' (pack_tc_head layout), bias rows, barriers,
  // TMEM (128 columns per group)
  {
    const uint4* src = a.wpack_tc + (int64_t)cw * (K::WB / 16);
    uint4* dst = reinterpret_cast<uint4*>(smem + offw);
    for (int k = threadIdx.x; k < K::WB / 16; k += blockDim.x) dst[k] = __ldg(src + k);
    const float* gb = a.bias + (int64_t)cw * H;
    for (int k = threadIdx.x; k < (M64 ? 64 : 32) * K::BR; k += blockDim.x) {
      const int m = k / K::BR, t = k % K::BR, h = m * S + t;
      bS[k] = (t < S && h < H) ? __ldg(gb + h) : 0.f;
    }
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < 8 + 16; k++) mbar_init(bars + k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t tcols = ngroups <= 1 ? 128u : (ngroups == 2 ? 256u : 512u);
  if (warp == 0) tmem_alloc(tmem_slot, tcols);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem0 = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const uint32_t tcol = tmem0 + 128u * (uint32_t)grp;
  const uint32_t tlane = (uint32_t)(32 * s) << 16;
  const bool mma_warp = s == 0;
  const uint32_t zt_s = smem_u32(zt), w_s = smem_u32(smem + offw);
  const float inv_sw = __ldg(a.wpack_inv_sw + cw);

  const int64_t cb0 = a.B * blockIdx.x / ctas_per_channel;
  const int64_t cb1 = a.B * (blockIdx.x + 1) / ctas_per_channel;
  const int64_t quads = (cb1 - cb0 + 3) / 4;
  const int64_t g0 = cb0 + 4 * (quads * grp / ngroups);
  const int64_t g1 = min(cb0 + 4 * (quads * (grp + 1) / ngroups), cb1);
  const int rounds = g1 > g0 ? (int)((g1 - g0 + 3) / 4) : 0;
  const int NS = N * S;
  const bool bulk = a.x_vec;   // every window start 16-byte aligned (and S % 4 == 0)
  const int64_t win0 = g0 + s;
  const float* xnext = a.x + win0 * a.xsb + c * a.xsc + a.r;
  float* ycur = a.y + (win0 * C + c) * H;
  const int64_t xstep = 4 * a.xsb, ystep = 4 * (int64_t)C * H;
  // segment row n of the series -> staging bytes n PITCH (bulk: one copy per row, or one copy
  // of the contiguous span when PITCH = 4 S; otherwise 4-byte cp.async per element)
  auto issue_load = [&](const float* xg) {
    if (bulk) {
      if constexpr (K::ROWCOPY) {
        if (lane == 0) mbar_arrive_expect(xbar, (uint32_t)NS * 4u);
        __syncwarp();
        if (lane < N)
          bulk_copy_nobar_expect(stage + lane * K::PITCH, xg + lane * S, 4u * S, xbar);
      } else {
        if (lane == 0) bulk_load(stage, xg, (uint32_t)NS * 4u, xbar);
      }
    } else {
      for (int k = lane; k < NS; k += 32) {
        const int n = k / S, t = k - n * S;
        cp_async4(stage + n * K::PITCH + 4 * t, xg + k);
      }
      cp_async_commit();
    }
  };

  uint32_t xph = 0, ph = 0;
  if (rounds > 0 && win0 < g1) {
    fence_proxy_async();
    issue_load(xnext);
  }
  const float4* xr4 = reinterpret_cast<const float4*>(stage + (valid ? i : N - 1) * K::PITCH);
  for (int rd = 0; rd < rounds; rd++) {
    const int64_t b = g0 + 4 * rd + s;
    const bool active = b < g1;
    float sx = 1.f, mi = 0.f, ki = 0.f, mu = 0.f;

    // ---------------- a1+a2: segment row i (Def 2) streamed from the staging area in three
    // passes: (A) sums of d = x - x0 and t~ d, (B) |z|^2 of z = d - mean d, (C) Z' rows
    if (active) {
      if (bulk) {
        mbar_wait_bounded(xbar, xph);
        xph ^= 1u;
      } else {
        cp_async_wait_all();
      }
      __syncwarp();
      const float x0 = reinterpret_cast<const float*>(xr4)[0];
      const float2 nx0 = f2(-x0);
      float2 s1a = f2(0.f), s1b = f2(0.f), s3a = f2(0.f), s3b = f2(0.f);
#pragma unroll
      for (int q = 0; q < K::NQ; q++) {
        const float4 v = xr4[q];
        const float2 d0 = add2(make_float2(v.x, v.y), nx0);
        const float2 d1 = add2(make_float2(v.z, v.w), nx0);
        s1a = add2(s1a, d0);
        s1b = add2(s1b, d1);
        s3a = fma2(make_float2(ttl<S>(4 * q), ttl<S>(4 * q + 1)), d0, s3a);
        s3b = fma2(make_float2(ttl<S>(4 * q + 2), ttl<S>(4 * q + 3)), d1, s3b);
      }
      const float2 s1 = add2(s1a, s1b), s3 = add2(s3a, s3b);
      const float m1 = (s1.x + s1.y) * a.inv_s;
      mu = x0 + m1;
      const float s3s = s3.x + s3.y;
      const float kap = s3s * a.inv_v;
      const float2 nm1 = f2(-m1);
      float2 qa = f2(0.f), qb = f2(0.f);
#pragma unroll
      for (int q = 0; q < K::NQ; q++) {
        const float4 v = xr4[q];
        const float2 z0 = add2(add2(make_float2(v.x, v.y), nx0), nm1);
        const float2 z1 = add2(add2(make_float2(v.z, v.w), nx0), nm1);
        qa = fma2(z0, z0, qa);
        qb = fma2(z1, z1, qb);
      }
      const float2 q2 = add2(qa, qb);
      const float nu2 = q2.x + q2.y;
      // Z' = z / sqrt(nu2 + eps_s) as split-fp16 rows [hi t | lo t], t >= S zero
      {
        const float zsc = valid ? rsqrtf(nu2 + kEpsSeasonal) : 0.f;
        const float2 zs2 = f2(zsc);
        const int r = 32 * s + i;
        unsigned char* zr = zt + (r >> 3) * K::SBO + (r & 7) * 16;
#pragma unroll
        for (int ch = 0; ch < K::SP / 8; ch++) {
          uint4 hv = make_uint4(0u, 0u, 0u, 0u), lv = make_uint4(0u, 0u, 0u, 0u);
          if (8 * ch < S) {
            const float4 v0 = xr4[2 * ch];
            const float2 z0 = mul2(add2(add2(make_float2(v0.x, v0.y), nx0), nm1), zs2);
            const float2 z1 = mul2(add2(add2(make_float2(v0.z, v0.w), nx0), nm1), zs2);
            split2(z0, hv.x, lv.x);
            split2(z1, hv.y, lv.y);
            if (8 * ch + 4 < S) {
              const float4 v1 = xr4[2 * ch + 1];
              const float2 z2 = mul2(add2(add2(make_float2(v1.x, v1.y), nx0), nm1), zs2);
              const float2 z3 = mul2(add2(add2(make_float2(v1.z, v1.w), nx0), nm1), zs2);
              split2(z2, hv.z, lv.z);
              split2(z3, hv.w, lv.w);
            }
          }
          sts128(zr + ch * 128, hv);
          sts128(zr + (K::SP / 8 + ch) * 128, lv);
        }
      }
      // |x_t| <= |mu| + |z|: the exact power-of-two scale of X'
      sx = pow2_scale(warp_max_nonneg(valid ? fabsf(mu) + fast_sqrt(nu2) : 0.f));
      // Def 5: sigma^2 = (1/(N S)) sum_n [nu2_n + S (mu_n - mubar)^2], both sums in one tree
      const float m0 = __shfl_sync(0xffffffffu, mu, 0);
      const float dd = valid ? mu - m0 : 0.f;
      float2 acc = make_float2(dd, valid ? fmaf((float)S * dd, dd, nu2) : 0.f);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        acc = add2(acc, make_float2(__shfl_xor_sync(0xffffffffu, acc.x, o),
                                    __shfl_xor_sync(0xffffffffu, acc.y, o)));
      const float var = fmaf(-(float)S * acc.x, acc.x * a.inv_n, acc.y) * a.inv_ns;
      // series-level factors by MUFU reciprocal / square root (<= ~1 ulp, a common relative
      // factor on every trend logit of the series)
      const float inv_var = fast_rcp(var + kEpsTrend);
      const float tsc = fast_sqrt(inv_var * a.kt);
      mi = mu * tsc;
      ki = kap * (tsc * fast_sqrt(a.vtrend));
      colv[i] = valid ? mi : INFINITY;
      colv[32 + i] = ki;
      colv[128 + i] = valid ? 0.f : -INFINITY;
      __syncwarp();
    }

    // ---------------- a3 Gram on tcgen05: rho = Z' Z'^T (4 series, diagonal blocks used):
    // hh, hl, lh as three runs of SP/16 K-steps
    fence_proxy_async();
    tc_fence_before();
    named_bar(1 + grp, 128);
    tc_fence_after();
    if (mma_warp && elect_one()) {
      constexpr uint32_t LO = (K::SP / 8) * 128;
#pragma unroll
      for (int k = 0; k < K::SP / 16; k++) {
        const uint32_t o = k * 256;
        umma(tcol, sdesc(zt_s + o, 128, K::SBO), sdesc(zt_s + o, 128, K::SBO), kIdGramG, k > 0);
        umma(tcol, sdesc(zt_s + o, 128, K::SBO), sdesc(zt_s + LO + o, 128, K::SBO), kIdGramG, true);
        umma(tcol, sdesc(zt_s + LO + o, 128, K::SBO), sdesc(zt_s + o, 128, K::SBO), kIdGramG, true);
      }
      umma_commit(mbar);
    }

    // ---------------- a4+a5 trend softmax (overlaps the Gram): lane j -> column j of A_t,
    // A_t[i][j] = E_ji / l_i (E symmetric, shift 0 = the row max at j = i)
    uint32_t th[16], tl[16];
    if (active) {
      float e[32];
      const float2 mi2 = f2(mi), ki2 = f2(ki);
      float2 sa = f2(0.f), sb = f2(0.f);
      const float4* cm4 = reinterpret_cast<const float4*>(colv);
      const float4* ck4 = reinterpret_cast<const float4*>(colv + 32);
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const float4 mj = cm4[q], kj = ck4[q];
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int j = 4 * q + 2 * h;
          const float2 dmj = add2(mi2, h ? make_float2(-mj.z, -mj.w) : make_float2(-mj.x, -mj.y));
          const float2 dkj = add2(ki2, h ? make_float2(-kj.z, -kj.w) : make_float2(-kj.x, -kj.y));
          const float2 ex =
              fma2(make_float2(-dkj.x, -dkj.y), dkj, mul2(make_float2(-dmj.x, -dmj.y), dmj));
          e[j] = fast_ex2(ex.x);
          e[j + 1] = fast_ex2(ex.y);
          if (h) sb = add2(sb, make_float2(e[j], e[j + 1]));
          else sa = add2(sa, make_float2(e[j], e[j + 1]));
        }
      }
      const float2 sum2 = add2(sa, sb);
      colv[64 + i] = valid ? fast_rcp(sum2.x + sum2.y) : 0.f;
      __syncwarp();
      const float4* cr4 = reinterpret_cast<const float4*>(colv + 64);
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const float4 r = cr4[q];
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int j = 4 * q + 2 * h;
          const float2 v = mul2(make_float2(e[j], e[j + 1]), h ? make_float2(r.z, r.w) : make_float2(r.x, r.y));
          if constexpr (DUMP) {   // v = (A_t[j][lane], A_t[j + 1][lane])
            if (valid) {
              float* d = a.a_t_dbg + (b * C + c) * (int64_t)N * N + lane;
              if (j < N) d[(int64_t)j * N] = v.x;
              if (j + 1 < N) d[(int64_t)(j + 1) * N] = v.y;
            }
          }
          split2(v, th[j / 2], tl[j / 2]);
        }
      }
    }

    // ---------------- Gram done: X' rows (x sx, split fp16) into this warp's quarter (its Z'
    // rows are read), then the staging area is free for the next series of this warp
    mbar_wait_bounded(mbar, ph);
    tc_fence_after();
    if (active) {
      const float xs = valid ? sx : 0.f;
      const float2 xs2 = f2(xs);
#pragma unroll
      for (int ch = 0; ch < K::NCT; ch++) {
        uint4 hv = make_uint4(0u, 0u, 0u, 0u), lv = make_uint4(0u, 0u, 0u, 0u);
        const float4 v0 = xr4[2 * ch];
        split2(mul2(make_float2(v0.x, v0.y), xs2), hv.x, lv.x);
        split2(mul2(make_float2(v0.z, v0.w), xs2), hv.y, lv.y);
        if (8 * ch + 4 < S) {
          const float4 v1 = xr4[2 * ch + 1];
          split2(mul2(make_float2(v1.x, v1.y), xs2), hv.z, lv.z);
          split2(mul2(make_float2(v1.z, v1.w), xs2), hv.w, lv.w);
        }
        unsigned char* p = xq + ch * 1024 + (i >> 3) * 128 + (i & 7) * 16;
        sts128(p, hv);
        sts128(p + 512, lv);
      }
      __syncwarp();
      xnext += xstep;
      if (b + 4 < g1) {
        fence_proxy_async();
        issue_load(xnext);
      }
    }

    // ---------------- a5 seasonal softmax from the Gram row in TMEM: lane j -> column j of
    // A_s, A_s[i][j] = F_ji / l_i, F = 2^((rho - 1) ks) (shift 1 >= rho, symmetric)
    if (active) {
      uint32_t sh[16], sl[16];
      {
        uint32_t gr[32];
        tld_x32(tcol + tlane + 32u * s, gr);
        tld_wait();
        float e[32];
        const float2 ks2 = f2(a.ks), nks2 = f2(-a.ks);
        const float4* cx4 = reinterpret_cast<const float4*>(colv + 128);
        float2 sa = f2(0.f), sb = f2(0.f);
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          float2 arg = fma2(make_float2(__uint_as_float(gr[j]), __uint_as_float(gr[j + 1])), ks2,
                            nks2);
          const float4 mk = cx4[j >> 2];
          arg = add2(arg, (j & 2) ? make_float2(mk.z, mk.w) : make_float2(mk.x, mk.y));
          e[j] = fast_ex2(arg.x);
          e[j + 1] = fast_ex2(arg.y);
          if (j & 2) sb = add2(sb, make_float2(e[j], e[j + 1]));
          else sa = add2(sa, make_float2(e[j], e[j + 1]));
        }
        const float2 sum2 = add2(sa, sb);
        colv[96 + i] = valid ? fast_rcp(sum2.x + sum2.y) : 0.f;
        __syncwarp();
        const float4* cr4 = reinterpret_cast<const float4*>(colv + 96);
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const float4 r = cr4[q];
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int j = 4 * q + 2 * h;
            const float2 v = mul2(make_float2(e[j], e[j + 1]), h ? make_float2(r.z, r.w) : make_float2(r.x, r.y));
            if constexpr (DUMP) {   // v = (A_s[j][lane], A_s[j + 1][lane])
              if (valid) {
                float* d = a.a_s_dbg + (b * C + c) * (int64_t)N * N + lane;
                if (j < N) d[(int64_t)j * N] = v.x;
                if (j + 1 < N) d[(int64_t)(j + 1) * N] = v.y;
              }
            }
            split2(v, sh[j / 2], sl[j / 2]);
          }
        }
      }
      // A^T rows into this warp's TMEM lanes (the Gram block is read): [0,16) A_s hi,
      // [16,32) A_t hi, [32,48) A_s lo, [48,64) A_t lo
      tst_x16(tcol + tlane, sh);
      tst_x16(tcol + tlane + 16u, th);
      tst_x16(tcol + tlane + 32u, sl);
      tst_x16(tcol + tlane + 48u, tl);
      tst_wait();
    }

    // ---------------- a6+a7 fold on tcgen05: Q'^T = [A_s^T | A_t^T] W'^T, D in [64, 96)
    tc_fence_before();
    named_bar(1 + grp, 128);
    tc_fence_after();
    if (mma_warp && elect_one()) {
#pragma unroll
      for (int ks = 0; ks < 4; ks++) {
        const uint64_t bh = sdesc(w_s + ks * 256, 128, 2048);
        const uint64_t bl = sdesc(w_s + (8 + 2 * ks) * 128, 128, 2048);
        const uint32_t idf = M64 ? kIdFoldG64 : (M <= 16 ? kIdFoldG16 : kIdFoldG);
        umma_ts(tcol + 64u, tcol + 8u * ks, bh, idf, ks > 0);
        umma_ts(tcol + 64u, tcol + 8u * ks, bl, idf, true);
        umma_ts(tcol + 64u, tcol + 32u + 8u * ks, bh, idf, true);
      }
      umma_commit(mbar + 1);
    }
    mbar_wait_bounded(mbar + 1, ph);
    tc_fence_after();

    // ---------------- a7 head on mma.sync, per warp: Y' = Q' X' (split fp16), Q' A-fragments
    // from TMEM (16x256b loads of Q'^T + movmatrix), X' B-fragments by ldmatrix.trans
    // M64: two passes of 32 future segments (Q'^T columns 64 + 32 mp)
#pragma unroll 1
    for (int mp = 0; mp < (M64 ? 2 : 1); mp++) {
    if (M64 && mp == 1 && M <= 32) break;
    if (active) {
      const int m0 = 32 * mp;
      const bool two_mt = M > m0 + 16;
      uint32_t qah[2][2][4], qal[2][2][4];   // [mt][kt][reg]
      if (!M64 && !two_mt) {
        // M <= 16 (one m-tile; the fold wrote 16 columns): the first two 8-column groups only
        uint32_t r0[8], r1[8];
        tld16_x2(tcol + ((uint32_t)(32 * s) << 16) + 64u, r0);
        tld16_x2(tcol + ((uint32_t)(32 * s + 16) << 16) + 64u, r1);
        tld_wait();
#pragma unroll
        for (int h = 0; h < 2; h++)
#pragma unroll
          for (int v = 0; v < 2; v++)
#pragma unroll
            for (int k = 0; k < 2; k++) {
              const uint32_t* r = h ? r1 : r0;
              uint32_t hi, lo;
              split2(make_float2(__uint_as_float(r[4 * k + 2 * v]), __uint_as_float(r[4 * k + 2 * v + 1])),
                     hi, lo);
              qah[0][h][(k & 1) + 2 * v] = movm_t(hi);
              qal[0][h][(k & 1) + 2 * v] = movm_t(lo);
            }
      } else {
        uint32_t r0[16], r1[16];
        tld16_x4(tcol + ((uint32_t)(32 * s) << 16) + 64u + 32u * mp, r0);
        tld16_x4(tcol + ((uint32_t)(32 * s + 16) << 16) + 64u + 32u * mp, r1);
        tld_wait();
#pragma unroll
        for (int h = 0; h < 2; h++)
#pragma unroll
          for (int v = 0; v < 2; v++)
#pragma unroll
            for (int k = 0; k < 4; k++) {
              const uint32_t* r = h ? r1 : r0;
              uint32_t hi, lo;
              split2(make_float2(__uint_as_float(r[4 * k + 2 * v]), __uint_as_float(r[4 * k + 2 * v + 1])),
                     hi, lo);
              qah[k >> 1][h][(k & 1) + 2 * v] = movm_t(hi);
              qal[k >> 1][h][(k & 1) + 2 * v] = movm_t(lo);
            }
      }
      const int l8 = lane & 7, g4 = lane >> 3;
      const float ys = inv_sw / sx;
      const float* bq = bS + 2 * (lane & 3);
      float* yg = ycur;
      const bool pairs = (H & 1) == 0;
      // n-tiles in groups of up to 4 (accumulators 2 x 4 x 4 registers)
      constexpr int NG = K::NCT < 4 ? K::NCT : 4;
#pragma unroll
      for (int n0 = 0; n0 < K::NCT; n0 += NG) {
        constexpr int dummy = 0;
        (void)dummy;
        float acc[2][NG][4];
#pragma unroll
        for (int mt = 0; mt < 2; mt++)
#pragma unroll
          for (int nt = 0; nt < NG; nt++)
#pragma unroll
            for (int e = 0; e < 4; e++) acc[mt][nt][e] = 0.f;
#pragma unroll
        for (int kt = 0; kt < 2; kt++) {
          uint32_t xh[NG][2], xl[NG][2];
#pragma unroll
          for (int nt = 0; nt < NG; nt += 2) {
            if (n0 + nt >= K::NCT) break;
            if (n0 + nt + 1 < K::NCT && nt + 1 < NG) {
              uint32_t r[4];
              const unsigned char* p =
                  xq + (n0 + nt + (g4 >> 1)) * 1024 + (2 * kt + (g4 & 1)) * 128 + l8 * 16;
              ldsm_x4_t(r, p);
              xh[nt][0] = r[0]; xh[nt][1] = r[1]; xh[nt + 1][0] = r[2]; xh[nt + 1][1] = r[3];
              ldsm_x4_t(r, p + 512);
              xl[nt][0] = r[0]; xl[nt][1] = r[1]; xl[nt + 1][0] = r[2]; xl[nt + 1][1] = r[3];
            } else {
              const unsigned char* p =
                  xq + (n0 + nt) * 1024 + (2 * kt + (g4 & 1)) * 128 + l8 * 16;
              ldsm_x2_t(xh[nt][0], xh[nt][1], p);
              ldsm_x2_t(xl[nt][0], xl[nt][1], p + 512);
            }
          }
#pragma unroll
          for (int mt = 0; mt < 2; mt++) {
            if (mt == 1 && !two_mt) break;
#pragma unroll
            for (int nt = 0; nt < NG; nt++)
              if (n0 + nt < K::NCT) mma16816_nv(acc[mt][nt], qal[mt][kt], xh[nt][0], xh[nt][1]);
#pragma unroll
            for (int nt = 0; nt < NG; nt++)
              if (n0 + nt < K::NCT) mma16816_nv(acc[mt][nt], qah[mt][kt], xl[nt][0], xl[nt][1]);
#pragma unroll
            for (int nt = 0; nt < NG; nt++)
              if (n0 + nt < K::NCT) mma16816_nv(acc[mt][nt], qah[mt][kt], xh[nt][0], xh[nt][1]);
          }
        }
        // ---------------- a8 store: y = Y' / (sw sx) + b (Def 11), pairs (m, t..t+1)
#pragma unroll
        for (int mt = 0; mt < 2; mt++) {
          if (mt == 1 && !two_mt) break;
#pragma unroll
          for (int hh = 0; hh < 2; hh++) {
            const int m = m0 + 16 * mt + 8 * hh + (lane >> 2);
            if (m >= M) continue;
#pragma unroll
            for (int nt = 0; nt < NG; nt++) {
              const int t = 8 * (n0 + nt) + 2 * (lane & 3);
              if (n0 + nt >= K::NCT || t >= S) continue;
              const int h = m * S + t;
              const float2 bb = *reinterpret_cast<const float2*>(bq + m * K::BR + 8 * (n0 + nt));
              const float ox = fmaf(acc[mt][nt][2 * hh], ys, bb.x);
              const float oy = fmaf(acc[mt][nt][2 * hh + 1], ys, bb.y);
              if (pairs && h + 1 < H) {
                asm volatile("st.global.cs.v2.f32 [%0], {%1,%2};" ::"l"(yg + h), "f"(ox), "f"(oy)
                             : "memory");
              } else {
                if (h < H) yg[h] = ox;
                if (h + 1 < H) yg[h + 1] = oy;
              }
            }
          }
        }
      }
    }
    }
    ph ^= 1u;
    ycur += ystep;
  }
  cp_async_wait_all();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem0, tcols);
}

namespace {
template <int S, bool M64>
int tcg_groups(int max_smem_optin) {
  using K = TcgCfg<S, M64>;
  int g = 4;
  while (g > 1 && (size_t)g * K::GROUP + K::FIXED > (size_t)max_smem_optin) g--;
  return (size_t)g * K::GROUP + K::FIXED <= (size_t)max_smem_optin ? g : 0;
}
template <int S, bool M64>
size_t tcg_smem(int g) {
  using K = TcgCfg<S, M64>;
  return (size_t)g * K::GROUP + K::FIXED;
}
}  // namespace

bool tcg_supported_s(int S) {
  return S == 12 || S == 16 || S == 32 || S == 48 || S == 64 || S == 96;
}

bool plan_tcg_kernel(const FwdArgs& a, int max_smem_optin, int sm_count, TcqPlan* p) {
  if (!tcg_supported_s(a.S) || a.N < 1 || a.N > 32 || a.M > 64) return false;
  const bool m64 = a.M > 32;
  int g = 0;
  size_t smem = 0;
  switch (a.S) {
#define PRNET_TCG_CASE(SV)                                                       \
  case SV:                                                                       \
    g = m64 ? tcg_groups<SV, true>(max_smem_optin) : tcg_groups<SV, false>(max_smem_optin); \
    smem = m64 ? tcg_smem<SV, true>(g) : tcg_smem<SV, false>(g);                 \
    break;
    PRNET_TCG_CASE(12)
    PRNET_TCG_CASE(16)
    PRNET_TCG_CASE(32)
    PRNET_TCG_CASE(48)
    PRNET_TCG_CASE(64)
    PRNET_TCG_CASE(96)
#undef PRNET_TCG_CASE
    default:
      return false;
  }
  if (g < 1) return false;
  p->groups = g;
  p->smem_bytes = smem;
  p->wins_per_group = 128;
  // one CTA per SM; split each channel into k CTAs against wave quantisation (as tc_quad)
  constexpr int64_t kPrologue = 32;
  const int64_t per_cta = (int64_t)g * p->wins_per_group;
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

template <int S, bool DUMP, bool M64>
static cudaError_t launch_tcg_t(const FwdArgs& a, const TcqPlan& p, cudaStream_t st) {
  auto k = prnet_fwd_tcg_kernel<S, DUMP, M64>;
  cudaError_t e =
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  const int64_t per_cta = (int64_t)p.groups * p.wins_per_group;
  const int ctas =
      p.ctas_per_channel > 0 ? p.ctas_per_channel : (int)((a.B + per_cta - 1) / per_cta);
  dim3 grid((unsigned)ctas, (unsigned)a.C);
  k<<<grid, 128 * p.groups, p.smem_bytes, st>>>(a, ctas);
  return cudaGetLastError();
}

cudaError_t launch_tcg_kernel(const FwdArgs& a, const TcqPlan& p, cudaStream_t st) {
  const bool dump = a.a_s_dbg != nullptr;
  switch (a.S) {
#define PRNET_TCG_L(SV) \
  case SV:              \
    if (a.M > 32)                                                                        \
      return dump ? launch_tcg_t<SV, true, true>(a, p, st) : launch_tcg_t<SV, false, true>(a, p, st); \
    return dump ? launch_tcg_t<SV, true, false>(a, p, st) : launch_tcg_t<SV, false, false>(a, p, st);
    PRNET_TCG_L(12)
    PRNET_TCG_L(16)
    PRNET_TCG_L(32)
    PRNET_TCG_L(48)
    PRNET_TCG_L(64)
    PRNET_TCG_L(96)
#undef PRNET_TCG_L
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace prnet
