// fwd_tc2.cu -- fused PRNet pattern-attention forward with EVERY contraction on the
// 5th-gen tensor cores (tcgen05.mma, accumulators in TMEM); S = 24, N <= 32, M <= 32.
//
// Same reading and split-fp16 3-product arithmetic as
// the other variants.  A CTA holds 3 independent groups of 4 warps; a group works
// on 4 series per round (warp w <-> series w <-> TMEM lanes 32w..32w+31):
//
//   a2   descriptors, lane i = segment i; Z' rows -> Gram tile (K-major),
//        X' rows -> head B tile (MN-major)                          [CUDA cores]
//   a3   Gram: for each series w, D[:, 32w..] += Z'(128 rows) Z'_w^T  [tcgen05, 24 MMA]
//   a4/5 trend softmax, lane-per-row (FA4 style: no shuffles), rows of A_t
//        -> fold A tile (MN-major)                                   [CUDA cores,
//                                                                      overlaps the Gram]
//   a5   tcgen05.ld of the series' 32x32 Gram block (lane = row i), seasonal
//        softmax lane-per-row -> fold A tile                         [CUDA cores]
//   a6/7 fold: Q'^T = [A_s^T | A_t^T] W'^T, W' (channel head) K-major  [tcgen05, 12 MMA]
//   a7   tcgen05.ld of Q'^T (lane = column j of Q'), split -> head A tile (MN-major);
//        head: for each w, D[:, 32w..] += Q'(128 rows) X'_w            [tcgen05, 24 MMA]
//   a8   tcgen05.ld of Y' (lane = future segment m, 24 values) -> y + b   [CUDA cores]
//
// The per-series Gram and head are block-diagonal on the M = 128 tile (each MMA's
// B operand is one series, so 3/4 of its rows are discarded): 4x the MACs of the
// product, paid on a unit that is 4x faster than mma.sync and issued by one
// thread, which is what removes the CUDA-core issue bottleneck of fwd_mma.cu.
//
// Per group: Gram/Q tile 16 KB, fold A tile 32 KB (also hosts the TMA staging of
// the next series), X' tile 16 KB; 3 groups + W' + bias ~= 209 KB; TMEM 3 x 160
// of 512 columns; 12 warps per SM.
#include <cuda_fp16.h>

#include <cmath>

#include "mma_common.cuh"

namespace prnet {

namespace {

__device__ __forceinline__ void tmem_alloc2(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
#define PRNET_LD_REGS16(r, o)                                                                  \
  "=r"(r[o + 0]), "=r"(r[o + 1]), "=r"(r[o + 2]), "=r"(r[o + 3]), "=r"(r[o + 4]),            \
      "=r"(r[o + 5]), "=r"(r[o + 6]), "=r"(r[o + 7]), "=r"(r[o + 8]), "=r"(r[o + 9]),        \
      "=r"(r[o + 10]), "=r"(r[o + 11]), "=r"(r[o + 12]), "=r"(r[o + 13]), "=r"(r[o + 14]),   \
      "=r"(r[o + 15])
// thread t of the warp <- TMEM lane (base lane + t), 32 / 16 / 8 consecutive fp32 columns
__device__ __forceinline__ void tld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : PRNET_LD_REGS16(r, 0), PRNET_LD_REGS16(r, 16)
      : "r"(taddr));
}
__device__ __forceinline__ void tld24(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : PRNET_LD_REGS16(r, 0)
      : "r"(taddr));
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23])
      : "r"(taddr + 16u));
}
__device__ __forceinline__ void tld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ void mbar_wait_to(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  uint64_t t0 = 0;
  for (uint32_t it = 0;; it++) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(20000u)   // suspend up to 20 us, no spinning
        : "memory");
    if (done) return;
    if ((it & 63u) == 0) {
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (it == 0) t0 = now;
      else if (now - t0 > 2000000000ull) __trap();
    }
  }
}
__device__ __forceinline__ void bar_group(uint32_t id) {
  asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory");
}
// 8 fp32 -> 16-byte hi and lo halves (v = hi + lo)
__device__ __forceinline__ void split8(const float* v, uint4& hi, uint4& lo) {
  uint32_t* h = reinterpret_cast<uint32_t*>(&hi);
  uint32_t* l = reinterpret_cast<uint32_t*>(&lo);
#pragma unroll
  for (int u = 0; u < 4; u++) split2(make_float2(v[2 * u], v[2 * u + 1]), h[u], l[u]);
}

}  // namespace

// ---- layout (bytes)
constexpr int kT2Groups = 3;
constexpr int kT2ZT = 16384;   // Gram operand tile (K-major, hi K 0..31, lo 32..63), later Q tile
constexpr int kT2AT = 32768;   // fold A tile (MN-major, K: s-hi 0..31, t-hi 32..63, s-lo, t-lo)
constexpr int kT2XT = 16384;   // head B tile (MN-major, N = t padded to 32, K = j: hi, lo)
constexpr int kT2Group = kT2ZT + kT2AT + kT2XT;
constexpr int kT2OffW = kT2Groups * kT2Group;        // W' (fold B operand), 8 KB
constexpr int kT2OffCol = kT2OffW + 8192;            // per warp: column vectors [4][32] fp32
constexpr int kT2OffBar = kT2OffCol + 12 * 512;      // mbarriers: 12 TMA + 3 x (G, F, H)
constexpr int kT2OffTmem = kT2OffBar + 24 * 8;
constexpr int kT2OffBias = kT2OffTmem + 64;
constexpr int kT2TmemCols = 512;

template <bool DBG>
__global__ void __launch_bounds__(384, 1) prnet_fwd_tc2_kernel(FwdArgs a, int wins_per_group) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int S = 24;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = warp >> 2, w = warp & 3;   // group, series slot in the group
  const int c = blockIdx.y;
  const int cw = a.head_per_channel ? c : 0;
  const int N = a.N, M = a.M, H = a.H, C = a.C;
  const int NS = N * S;
  const int i = lane;

  unsigned char* gbase = smem + grp * kT2Group;
  unsigned char* ztile = gbase;                   // Gram operand, later the head's Q tile
  unsigned char* atile = gbase + kT2ZT;           // fold A tile
  unsigned char* xtile = gbase + kT2ZT + kT2AT;   // head B tile
  unsigned char* wsm = smem + kT2OffW;
  float* xbuf = reinterpret_cast<float*>(atile + w * 8192);   // TMA staging in the warp's slice
  float* colv = reinterpret_cast<float*>(smem + kT2OffCol + warp * 512);  // [4][32]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kT2OffBar);
  uint64_t* xbar = bars + warp;
  uint64_t* gbar = bars + 12 + 3 * grp;   // Gram, fold, head completion
  uint32_t* tmem_s = reinterpret_cast<uint32_t*>(smem + kT2OffTmem);
  float* bS = reinterpret_cast<float*>(smem + kT2OffBias);

  // ---------------- prologue: channel head, zero padding, barriers, TMEM
  const float inv_sw = a.wpack_inv_sw[cw];
  {
    const uint4* src = a.wpack_tc + (int64_t)cw * (8192 / 16);
    uint4* dst = reinterpret_cast<uint4*>(wsm);
    for (int k = threadIdx.x; k < 8192 / 16; k += blockDim.x) dst[k] = __ldg(src + k);
    const float* gb = a.bias + (int64_t)cw * H;
    for (int k = threadIdx.x; k < H; k += blockDim.x) bS[k] = __ldg(gb + k);
    // all three tiles of every group start at zero (X' padding rows / t >= 24 stay zero)
    uint4* z = reinterpret_cast<uint4*>(smem);
    for (int k = threadIdx.x; k < kT2Groups * kT2Group / 16; k += blockDim.x)
      z[k] = make_uint4(0, 0, 0, 0);
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < 21; k++) mbar_init(bars + k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc2(tmem_s, kT2TmemCols);
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tmem_s + 160u * grp;        // G / Y blocks at +32w, Q at +128
  const uint32_t tlane = (uint32_t)(32 * w) << 16;    // this warp's TMEM lanes

  // instruction descriptors: D f32; A, B f16; N = 32; M = 128; majors per operand
  constexpr uint32_t kBase = (1u << 4) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
  constexpr uint32_t kIdGram = kBase;                              // A K-major, B K-major
  constexpr uint32_t kIdFold = kBase | (1u << 15);                 // A MN-major, B K-major
  constexpr uint32_t kIdHead = kBase | (1u << 15) | (1u << 16);    // A MN-major, B MN-major
  const uint32_t z_s = smem_u32(ztile), a_s = smem_u32(atile), x_s = smem_u32(xtile),
                 w_s = smem_u32(wsm);
  const bool leader = (w == 0) && (lane == 0);

  // windows: this group handles [g_begin, g_end), 4 per round
  const int64_t b_block = (int64_t)blockIdx.x * (kT2Groups * wins_per_group);
  const int64_t g_begin = b_block + (int64_t)grp * wins_per_group;
  int64_t g_end = g_begin + wins_per_group;
  if (g_end > a.B) g_end = a.B;
  const int rounds = g_end > g_begin ? (int)((g_end - g_begin + 3) / 4) : 0;
  const bool vec_x = a.x_vec && ((NS & 3) == 0);
  uint32_t xphase = 0, rphase = 0;

  auto issue_load = [&](int64_t bb) {
    const float* xg = a.x + bb * a.xsb + c * a.xsc + a.r;
    if (vec_x) {
      if (lane == 0) bulk_load(xbuf, xg, (uint32_t)NS * 4u, xbar);
    } else {
      for (int k = lane; k < NS; k += 32) cp_async4(xbuf + k, xg + k);
      cp_async_commit();
    }
  };

  if (g_begin + w < g_end) issue_load(g_begin + w);
  for (int rd = 0; rd < rounds; rd++) {
    const int64_t b = g_begin + 4 * rd + w;
    const bool active = b < g_end;
    const int64_t series = b * C + c;
    float sx = 1.f;
    float mu = 0.f, kap = 0.f, nu2 = 0.f, sz = 1.f;

    // ---------------- a2: descriptors (Def 4-5), lane i = segment i (registers)
    if (active) {
      if (vec_x) {
        mbar_wait_to(xbar, xphase);
        xphase ^= 1u;
      } else {
        cp_async_wait_all();
      }
      __syncwarp();
      float xv[24];
      float x0 = 0.f, m1 = 0.f;
      float2 s1 = f2(0.f), s3 = f2(0.f);
      float amx = 0.f, dmx = 0.f;
      const int row = i < N ? i : 0;   // lanes past N mirror row 0 (results masked)
      const float4* xr = reinterpret_cast<const float4*>(xbuf + row * 24);
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
      sx = pow2_scale(warp_max(amx));
      sz = pow2_scale(2.f * warp_max(dmx));
      float zv[24];
      float2 q2 = f2(0.f);
      {
        const float2 nx0 = f2(-x0), nm1 = f2(-m1), sz2 = f2(sz), sx2 = f2(sx);
#pragma unroll
        for (int t = 0; t < 24; t += 2) {
          const float2 z = add2(add2(make_float2(xv[t], xv[t + 1]), nx0), nm1);
          q2 = fma2(z, z, q2);
          const float2 zs = mul2(z, sz2), xs = mul2(make_float2(xv[t], xv[t + 1]), sx2);
          zv[t] = zs.x;
          zv[t + 1] = zs.y;
          xv[t] = xs.x;
          xv[t + 1] = xs.y;
        }
      }
      nu2 = q2.x + q2.y;
      if (i < N) {
        // Z' row i -> Gram tile (K-major; row r = 32w + i: (r/8)*1024 + kc*128 + (r%8)*16),
        // K chunks 0..2 hi, 4..6 lo; chunks 3, 7 (t = 24..31) are the zero K padding
        unsigned char* zr = ztile + (4 * w + (i >> 3)) * 1024 + (i & 7) * 16;
#pragma unroll
        for (int q = 0; q < 3; q++) {
          uint4 h, l;
          split8(zv + 8 * q, h, l);
          *reinterpret_cast<uint4*>(zr + q * 128) = h;
          *reinterpret_cast<uint4*>(zr + (4 + q) * 128) = l;
        }
        *reinterpret_cast<uint4*>(zr + 3 * 128) = make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(zr + 7 * 128) = make_uint4(0, 0, 0, 0);
        // X' row j = i -> head B tile (MN-major, N = t: (t/8)*1024 + kc*128 + (j%8)*16),
        // K chunk j/8 (hi) and 4 + j/8 (lo)
        unsigned char* xr2 = xtile + w * 4096 + (i >> 3) * 128 + (i & 7) * 16;
#pragma unroll
        for (int q = 0; q < 3; q++) {
          uint4 h, l;
          split8(xv + 8 * q, h, l);
          *reinterpret_cast<uint4*>(xr2 + q * 1024) = h;
          *reinterpret_cast<uint4*>(xr2 + q * 1024 + 4 * 128) = l;
        }
      } else {
        // padding rows of the Gram tile must be zero (the tile was the Q tile last round)
        unsigned char* zr = ztile + (4 * w + (i >> 3)) * 1024 + (i & 7) * 16;
#pragma unroll
        for (int q = 0; q < 8; q++) *reinterpret_cast<uint4*>(zr + q * 128) = make_uint4(0, 0, 0, 0);
      }
    } else {
      // idle slot: its Gram rows must not be NaN (they only feed discarded outputs)
      unsigned char* zr = ztile + (4 * w + (i >> 3)) * 1024 + (i & 7) * 16;
#pragma unroll
      for (int q = 0; q < 8; q++) *reinterpret_cast<uint4*>(zr + q * 128) = make_uint4(0, 0, 0, 0);
    }
    // Def 5: sigma^2 = (1/(N S)) sum_n [nu2_n + S (mu_n - mubar)^2]
    const float mbar_ = warp_sum(i < N ? mu : 0.f) * a.inv_n;
    const float dv = i < N ? nu2 + (float)S * (mu - mbar_) * (mu - mbar_) : 0.f;
    const float inv_var = 1.0f / (warp_sum(dv) * a.inv_ns + kEpsTrend);
    const float inv = i < N ? rsqrtf(nu2 + kEpsSeasonal) : 0.f;
    const float cmt = sqrtf(inv_var * a.kt), ckt = sqrtf(a.vtrend * inv_var * a.kt);
    const float mus = i < N ? mu * cmt : 0.f, kas = i < N ? kap * ckt : 0.f;
    // column vectors for the lane-per-row softmaxes (broadcast reads)
    colv[i] = inv;                               // 0 past N
    colv[32 + i] = i < N ? 0.f : -INFINITY;      // additive mask
    colv[64 + i] = i < N ? mus : INFINITY;       // trend: +inf -> exponent -inf past N
    colv[96 + i] = kas;
    __syncwarp();

    // ---------------- a3 Gram on tcgen05 (series w' block into D columns 32 w')
    fence_async_smem();
    fence_before();
    bar_group(1 + grp);
    fence_after();
    if (leader) {
#pragma unroll
      for (int ws = 0; ws < 4; ws++) {
#pragma unroll
        for (int ks = 0; ks < 2; ks++) {
          const uint64_t ah = sdesc(z_s + ks * 256, 128, 1024);
          const uint64_t al = sdesc(z_s + (4 + 2 * ks) * 128, 128, 1024);
          const uint64_t bh = sdesc(z_s + ws * 4096 + ks * 256, 128, 1024);
          const uint64_t bl = sdesc(z_s + ws * 4096 + (4 + 2 * ks) * 128, 128, 1024);
          const uint32_t d = tbase + 32u * ws;
          umma_f16(d, ah, bh, kIdGram, ks > 0 ? 1u : 0u);
          umma_f16(d, ah, bl, kIdGram, 1u);
          umma_f16(d, al, bh, kIdGram, 1u);
        }
      }
      umma_commit(gbar);
    }

    // A tile rows: k-row kk (K index), 4 chunks of 8 j's: (4w + jc)*2048 + (kk/8)*128 + (kk%8)*16
    unsigned char* arow = atile + w * 8192 + (i & 7) * 16;
    const int kc_i = i >> 3;

    // ---------------- a4+a5 trend softmax, row i (Def 7-8): exponent
    // -(mu~_i - mu~_j)^2 - (k~_i - k~_j)^2, row max 0 at j = i  -> K 32.. (hi), 96.. (lo)
    if (active) {
      const float4* cm4 = reinterpret_cast<const float4*>(colv + 64);
      const float4* ck4 = reinterpret_cast<const float4*>(colv + 96);
      float e[32];
      float2 sum2 = f2(0.f);
      const float2 mi = f2(mus), ki = f2(kas);
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const float4 mj = cm4[q], kj = ck4[q];
        const float2 dm0 = add2(mi, make_float2(-mj.x, -mj.y)), dm1 = add2(mi, make_float2(-mj.z, -mj.w));
        const float2 dk0 = add2(ki, make_float2(-kj.x, -kj.y)), dk1 = add2(ki, make_float2(-kj.z, -kj.w));
        const float2 a0 = fma2(make_float2(-dk0.x, -dk0.y), dk0, mul2(make_float2(-dm0.x, -dm0.y), dm0));
        const float2 a1 = fma2(make_float2(-dk1.x, -dk1.y), dk1, mul2(make_float2(-dm1.x, -dm1.y), dm1));
        e[4 * q] = fast_ex2(a0.x);
        e[4 * q + 1] = fast_ex2(a0.y);
        e[4 * q + 2] = fast_ex2(a1.x);
        e[4 * q + 3] = fast_ex2(a1.y);
        sum2 = add2(sum2, add2(make_float2(e[4 * q], e[4 * q + 1]), make_float2(e[4 * q + 2], e[4 * q + 3])));
      }
      const float rs = i < N ? 1.f / (sum2.x + sum2.y) : 0.f;
      const float2 rs2 = f2(rs);
#pragma unroll
      for (int q = 0; q < 16; q++) {
        const float2 p = mul2(make_float2(e[2 * q], e[2 * q + 1]), rs2);
        e[2 * q] = p.x;
        e[2 * q + 1] = p.y;
      }
      if constexpr (DBG) {
        if (i < N)
          for (int j = 0; j < N; j++) a.a_t_dbg[(series * N + i) * N + j] = e[j];
      }
#pragma unroll
      for (int jc = 0; jc < 4; jc++) {
        uint4 h, l;
        split8(e + 8 * jc, h, l);
        *reinterpret_cast<uint4*>(arow + jc * 2048 + (4 + kc_i) * 128) = h;
        *reinterpret_cast<uint4*>(arow + jc * 2048 + (12 + kc_i) * 128) = l;
      }
    }

    // ---------------- a5 seasonal softmax, row i (Def 6, 8): rho_ij = G'_ij inv_i inv_j / sz^2
    mbar_wait_to(gbar, rphase);
    fence_after();
    {
      uint32_t gr[32];
      tld32(tbase + tlane + 32u * w, gr);
      tld_wait();
      if (active) {
        const float4* ci4 = reinterpret_cast<const float4*>(colv);
        const float4* cx4 = reinterpret_cast<const float4*>(colv + 32);
        float u[32];
        float mx = -INFINITY;
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const float4 cv = ci4[q], mk = cx4[q];
          const float2 u0 = fma2(make_float2(__uint_as_float(gr[4 * q]), __uint_as_float(gr[4 * q + 1])),
                                 make_float2(cv.x, cv.y), make_float2(mk.x, mk.y));
          const float2 u1 = fma2(make_float2(__uint_as_float(gr[4 * q + 2]), __uint_as_float(gr[4 * q + 3])),
                                 make_float2(cv.z, cv.w), make_float2(mk.z, mk.w));
          u[4 * q] = u0.x;
          u[4 * q + 1] = u0.y;
          u[4 * q + 2] = u1.x;
          u[4 * q + 3] = u1.y;
          mx = fmaxf(mx, fmaxf(fmaxf(u0.x, u0.y), fmaxf(u1.x, u1.y)));
        }
        const float rk = (i < N ? inv : 1.f) * a.ks / (sz * sz);
        const float2 rk2 = f2(rk), nb2 = f2(-mx * rk);
        float2 sum2 = f2(0.f);
#pragma unroll
        for (int q = 0; q < 16; q++) {
          const float2 arg = fma2(make_float2(u[2 * q], u[2 * q + 1]), rk2, nb2);
          u[2 * q] = fast_ex2(arg.x);
          u[2 * q + 1] = fast_ex2(arg.y);
          sum2 = add2(sum2, make_float2(u[2 * q], u[2 * q + 1]));
        }
        const float2 rs2 = f2(i < N ? 1.f / (sum2.x + sum2.y) : 0.f);
#pragma unroll
        for (int q = 0; q < 16; q++) {
          const float2 p = mul2(make_float2(u[2 * q], u[2 * q + 1]), rs2);
          u[2 * q] = p.x;
          u[2 * q + 1] = p.y;
        }
        if constexpr (DBG) {
          if (i < N)
            for (int j = 0; j < N; j++) a.a_s_dbg[(series * N + i) * N + j] = u[j];
        }
#pragma unroll
        for (int jc = 0; jc < 4; jc++) {
          uint4 h, l;
          split8(u + 8 * jc, h, l);
          *reinterpret_cast<uint4*>(arow + jc * 2048 + kc_i * 128) = h;
          *reinterpret_cast<uint4*>(arow + jc * 2048 + (8 + kc_i) * 128) = l;
        }
      }
    }

    // ---------------- a6+a7 fold on tcgen05: Q'^T[(w, j)][m] -> D columns 128..159
    fence_async_smem();
    fence_before();
    bar_group(1 + grp);
    fence_after();
    if (leader) {
#pragma unroll
      for (int ks = 0; ks < 4; ks++) {
        const uint64_t ah = sdesc(a_s + ks * 256, 128, 2048);
        const uint64_t al = sdesc(a_s + (8 + 2 * ks) * 128, 128, 2048);
        const uint64_t bh = sdesc(w_s + ks * 256, 128, 2048);
        const uint64_t bl = sdesc(w_s + (8 + 2 * ks) * 128, 128, 2048);
        umma_f16(tbase + 128u, ah, bh, kIdFold, ks > 0 ? 1u : 0u);
        umma_f16(tbase + 128u, ah, bl, kIdFold, 1u);
        umma_f16(tbase + 128u, al, bh, kIdFold, 1u);
      }
      umma_commit(gbar + 1);
    }
    mbar_wait_to(gbar + 1, rphase);
    fence_after();
    {
      uint32_t qr[32];
      tld32(tbase + tlane + 128u, qr);   // lane j: Q'[m][j], m = 0..31
      tld_wait();
      // the A tile is consumed: stage the next series into this warp's slice
      const int64_t bn = b + 4;
      if (bn < g_end) issue_load(bn);
      // Q' column j -> head A tile (MN-major, M = (w, m), K = j): (4w + mc)*1024 +
      // (j/8)*128 (+512 lo) + (j%8)*16; rows j >= N are zero because A's columns are
      unsigned char* qrow = ztile + 4 * w * 1024 + (i >> 3) * 128 + (i & 7) * 16;
#pragma unroll
      for (int mc = 0; mc < 4; mc++) {
        float qv[8];
#pragma unroll
        for (int u = 0; u < 8; u++) qv[u] = __uint_as_float(qr[8 * mc + u]);
        uint4 h, l;
        split8(qv, h, l);
        *reinterpret_cast<uint4*>(qrow + mc * 1024) = h;
        *reinterpret_cast<uint4*>(qrow + mc * 1024 + 512) = l;
      }
    }

    // ---------------- a7 head on tcgen05: Y'_w' = Q'_w' X'_w' -> D columns 32 w'
    fence_async_smem();
    fence_before();
    bar_group(1 + grp);
    fence_after();
    if (leader) {
#pragma unroll
      for (int ws = 0; ws < 4; ws++) {
#pragma unroll
        for (int ks = 0; ks < 2; ks++) {
          const uint64_t ah = sdesc(z_s + ks * 256, 128, 1024);
          const uint64_t al = sdesc(z_s + (4 + 2 * ks) * 128, 128, 1024);
          const uint64_t bh = sdesc(x_s + ws * 4096 + ks * 256, 128, 1024);
          const uint64_t bl = sdesc(x_s + ws * 4096 + (4 + 2 * ks) * 128, 128, 1024);
          const uint32_t d = tbase + 32u * ws;
          umma_f16(d, ah, bh, kIdHead, ks > 0 ? 1u : 0u);
          umma_f16(d, ah, bl, kIdHead, 1u);
          umma_f16(d, al, bh, kIdHead, 1u);
        }
      }
      umma_commit(gbar + 2);
    }
    mbar_wait_to(gbar + 2, rphase);
    fence_after();

    // ---------------- a8 store: lane m holds Y'[m][0..23]; y = Y' / (sw sx) + b
    {
      uint32_t yr[32];
      tld24(tbase + tlane + 32u * w, yr);
      tld_wait();
      const int m = lane;
      if (active && m < M) {
        const float2 ys2 = f2(inv_sw / sx);
        float* yg = a.y + series * H + m * 24;
        const float* bm = bS + m * 24;
        if ((H % 24) == 0 && (H & 3) == 0) {
#pragma unroll
          for (int q = 0; q < 6; q++) {
            const float4 bb = *reinterpret_cast<const float4*>(bm + 4 * q);
            const float2 o0 = fma2(make_float2(__uint_as_float(yr[4 * q]), __uint_as_float(yr[4 * q + 1])), ys2,
                                   make_float2(bb.x, bb.y));
            const float2 o1 = fma2(make_float2(__uint_as_float(yr[4 * q + 2]), __uint_as_float(yr[4 * q + 3])),
                                   ys2, make_float2(bb.z, bb.w));
            stg_stream4(yg + 4 * q, make_float4(o0.x, o0.y, o1.x, o1.y));
          }
        } else {
          for (int t = 0; t < 24; t++) {
            if (m * 24 + t < H) yg[t] = __uint_as_float(yr[t]) * ys2.x + bm[t];
          }
        }
      }
    }
    rphase ^= 1u;
    fence_before();
  }
  cp_async_wait_all();
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc2(*tmem_s, kT2TmemCols);
}

bool plan_tc2_kernel(const FwdArgs& a, int max_smem_optin, Tc2Plan* p) {
  if (a.S != 24 || a.N > 32 || a.M > 32) return false;
  p->smem_bytes = (size_t)kT2OffBias + (size_t)a.H * 4;
  if (p->smem_bytes > (size_t)max_smem_optin) return false;
  p->wins_per_group = 32;
  return true;
}

template <bool DBG>
static cudaError_t launch_tc2_t(const FwdArgs& a, const Tc2Plan& p, cudaStream_t st) {
  auto k = prnet_fwd_tc2_kernel<DBG>;
  cudaError_t e =
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  const int64_t per_cta = (int64_t)kT2Groups * p.wins_per_group;
  dim3 grid((unsigned)((a.B + per_cta - 1) / per_cta), (unsigned)a.C);
  k<<<grid, 32 * 4 * kT2Groups, p.smem_bytes, st>>>(a, p.wins_per_group);
  return cudaGetLastError();
}

cudaError_t launch_tc2_kernel(const FwdArgs& a, const Tc2Plan& p, cudaStream_t st) {
  return a.a_s_dbg != nullptr ? launch_tc2_t<true>(a, p, st) : launch_tc2_t<false>(a, p, st);
}

}  // namespace prnet
