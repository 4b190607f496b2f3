// fwd_tc.cu -- fused PRNet pattern-attention forward with the fold on the 5th-gen
// tensor cores (tcgen05.mma, accumulator in TMEM); S = 24, 16 < N <= 32, M <= 32.
//
// Same per-series step map and reading as fwd_warp.cu / fwd_mma.cu
// and the same split-fp16 3-product arithmetic.  What changes is
// where the one dense contraction with a shared operand runs:
//
//   a6+a7 fold   Q^T = [A_s^T | A_t^T] [W_s | W_t]^T    (per channel W shared by
//                all series of the CTA)
//
// A CTA is one group of 4 warps, warp w owning one series per round.  Each warp
// computes its series' Gram (mma.sync, registers) and both row softmaxes on the
// accumulator fragments, and writes the attention tiles straight from the
// fragments into ITS 32-row slice of the CTA's 128 x 128 fp16 A tile (hi in K
// columns 0..63, lo in 64..127; MN-major canonical layout, so one fragment
// register is one 32-bit word of a core matrix and a warp store fills 128
// contiguous bytes).  One elected thread then issues 12 tcgen05.mma
// (M = 128 = 4 series x 32 rows, N = 32 future segments, K = 4 x 16) with the
// channel's W' (K-major, pre-packed at load time) as B, accumulating
// hi*hi + hi*lo + lo*hi in a 32-column TMEM accumulator, and commits to an
// mbarrier.  Each warp reads its 32 TMEM lanes back (tcgen05.ld 32x32b: lane j
// = row j of Q^T), splits Q into hi/lo through shared memory and runs the
// per-series head Y = Q X on mma.sync as in fwd_mma.cu.
//
// The per-series Gram and head stay on mma.sync: tcgen05 prices M = 64 like
// M = 128, so a 32 x 32 per-series product would be block-diagonal at 4x
// waste.
//
// Shared memory per CTA (4 warps): A tile 32 KB (each warp's 8 KB slice also
// hosts its TMA staging buffer, its fp16 Z and its fp16 Q staging at disjoint
// times), X' 4 x 3 KB, W' 8 KB, bias, barriers -> ~55 KB: 4 CTAs / 16 warps per
// SM; TMEM 32 columns per CTA.
#include <cuda_fp16.h>

#include <cmath>

#include "mma_common.cuh"

namespace prnet {

namespace {

// ---- tcgen05 / TMEM wrappers (PTX ISA 8.7, sm_100a)
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem desc] * B[smem desc], kind::f16 (fp16 in, fp32 accumulate)
__device__ __forceinline__ void tc_mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
// 32 lanes x 32 consecutive fp32 columns: thread t gets row (lane base + t)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int k = 0; k < 32; k++) v[k] = __uint_as_float(r[k]);
}
// Shared-memory matrix descriptor, SWIZZLE_NONE canonical layout (version 1 = sm100):
// start >> 4 at [0,14), LBO >> 4 at [16,30), SBO >> 4 at [32,46), version at [46,48).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
// Bounded mbarrier wait: a lost arrival traps (kernel error) after ~2 s instead of
// hanging the device.
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  uint64_t t0 = 0;
  for (uint32_t it = 0;; it++) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if ((it & 1023u) == 0) {
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (it == 0) t0 = now;
      else if (now - t0 > 2000000000ull) __trap();
    }
  }
}
__device__ __forceinline__ void group_bar(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace

// ---- layout constants (bytes)
constexpr int kTcWarps = 4;
constexpr int kTcSlice = 8192;                    // per-warp A slice: 32 rows x 128 K fp16
constexpr int kTcATile = kTcWarps * kTcSlice;     // 32 KB, M-chunk stride (SBO) 2048 B
constexpr int kTcXs = 32 * 24 * 2;                // X' hi (or lo): 32 rows x 24 halves
constexpr int kTcXRegion = 2 * kTcXs;             // X' hi + lo per warp
constexpr int kTcOffX = kTcATile;
constexpr int kTcOffW = kTcOffX + kTcWarps * kTcXRegion;   // W' B operand, 8 KB
constexpr int kTcWBytes = 4 * 2048;
constexpr int kTcOffMisc = kTcOffW + kTcWBytes;             // barriers, tmem address
constexpr int kTcOffBias = kTcOffMisc + 128;
// inside a slice (disjoint in time, see header): TMA staging fp32 [30..32][24] at 0,
// Z' hi/lo [32][24] and later Q' staging hi/lo [32][40] at 2880..
constexpr int kTcSlZ = 3072;
constexpr int kTcSlQ = 3072;
constexpr int kTcQRow = 80;   // bytes per Q' staging row (32 halves + 16 B pad)

int tc_wpack_bytes() { return kTcWBytes; }

// W' as the K-major B operand: element (m, k) at (m/8)*2048 + (k/8)*128 + (m%8)*16 + (k%8)*2,
// k = i (seasonal, 0..31) | 32 + i (trend) for hi, and +64 for lo.
void pack_tc_head(const float* ws, const float* wt, int Cw, int M, int N, unsigned char* out,
                  float* inv_sw) {
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
    __half* dst = reinterpret_cast<__half*>(out + (size_t)c * kTcWBytes);
    for (int m = 0; m < 32; m++)
      for (int k = 0; k < 64; k++) {
        float v = 0.f;
        if (m < M) {
          if (k < 32) {
            if (k < N) v = s[m * N + k] * sw;
          } else if (k - 32 < N) {
            v = t[m * N + (k - 32)] * sw;
          }
        }
        const __half h = __float2half_rn(v);
        const __half l = __float2half_rn(v - __half2float(h));
        const int kh = k, kl = 64 + k;
        dst[((m / 8) * 2048 + (kh / 8) * 128 + (m % 8) * 16 + (kh % 8) * 2) / 2] = h;
        dst[((m / 8) * 2048 + (kl / 8) * 128 + (m % 8) * 16 + (kl % 8) * 2) / 2] = l;
      }
  }
}

template <int MMT, bool DBG>
__global__ void __launch_bounds__(128, 4) prnet_fwd_tc_kernel(FwdArgs a, int wins_per_cta) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int MT = 2, S = 24;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, cq = lane & 3, q8 = lane >> 3;
  const int c = blockIdx.y;
  const int cw = a.head_per_channel ? c : 0;
  const int N = a.N, M = a.M, H = a.H, C = a.C;
  const int NS = N * S;

  unsigned char* atile = smem;
  unsigned char* slice = smem + warp * kTcSlice;
  float* xbuf = reinterpret_cast<float*>(slice);
  __half* z_hi = reinterpret_cast<__half*>(slice + kTcSlZ);
  __half* z_lo = z_hi + 32 * 24;
  unsigned char* qst = slice + kTcSlQ;   // Q' staging [j][m] hi rows, then lo rows
  __half* x_hi = reinterpret_cast<__half*>(smem + kTcOffX + warp * kTcXRegion);
  __half* x_lo = x_hi + 32 * 24;
  unsigned char* wsm = smem + kTcOffW;
  uint64_t* xbar = reinterpret_cast<uint64_t*>(smem + kTcOffMisc) + warp;   // TMA, per warp
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + kTcOffMisc) + 4;      // MMA commit
  uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(smem + kTcOffMisc + 64);
  float* bS = reinterpret_cast<float*>(smem + kTcOffBias);

  // ---------------- prologue: head of channel c (W' B operand + bias), barriers, TMEM
  const float inv_sw = a.wpack_inv_sw[cw];
  {
    const uint4* src = a.wpack_tc + (int64_t)cw * (kTcWBytes / 16);
    uint4* dst = reinterpret_cast<uint4*>(wsm);
    for (int k = threadIdx.x; k < kTcWBytes / 16; k += blockDim.x) dst[k] = __ldg(src + k);
    const float* gb = a.bias + (int64_t)cw * H;
    for (int k = threadIdx.x; k < H; k += blockDim.x) bS[k] = __ldg(gb + k);
    // X' padding rows (>= N) stay zero
    uint32_t* px = reinterpret_cast<uint32_t*>(x_hi);
    for (int k = lane; k < kTcXRegion / 4; k += 32) px[k] = 0u;
  }
  if (threadIdx.x == 0) {
    for (int w = 0; w < 4; w++) mbar_init(reinterpret_cast<uint64_t*>(smem + kTcOffMisc) + w, 1);
    mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tmem_base_s, 32);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // W' visible to the MMA
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_d = *tmem_base_s;

  // instruction descriptor: D f32 (bits 4-5 = 1), A/B f16, A MN-major (bit 15),
  // B K-major, N = 32 (bits 17-22 = N >> 3), M = 128 (bits 24-28 = M >> 4)
  constexpr uint32_t kIdesc = (1u << 4) | (1u << 15) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
  const uint32_t a_base = smem_u32(atile), w_base = smem_u32(wsm);

  const int64_t b_begin = (int64_t)blockIdx.x * wins_per_cta;
  int64_t b_end = b_begin + wins_per_cta;
  if (b_end > a.B) b_end = a.B;
  const int rounds = (int)((b_end - b_begin + 3) / 4);
  const bool vec_x = a.x_vec && ((NS & 3) == 0);
  uint32_t xphase = 0, mphase = 0;

  auto issue_load = [&](int64_t bb) {
    const float* xg = a.x + bb * a.xsb + c * a.xsc + a.r;
    if (vec_x) {
      if (lane == 0) bulk_load(xbuf, xg, (uint32_t)NS * 4u, xbar);
    } else {
      for (int k = lane; k < NS; k += 32) cp_async4(xbuf + k, xg + k);
      cp_async_commit();
    }
  };

  if (b_begin + warp < b_end) issue_load(b_begin + warp);
  for (int rd = 0; rd < rounds; rd++) {
    const int64_t b = b_begin + 4 * rd + warp;
    const bool active = b < b_end;
    const int64_t series = b * C + c;
    float nu2 = 0.f, mu = 0.f, kap = 0.f, sx = 1.f, sz = 1.f;
    const int i = lane;
    float g[MT][2 * MT][4];
    if (active) {
      if (vec_x) {
        mbar_wait_bounded(xbar, xphase);
        xphase ^= 1u;
      } else {
        cp_async_wait_all();
      }
      __syncwarp();

      // ---------------- a2: descriptors (Def 4-5), lane i = segment i (registers)
      float xv[24];
      float x0 = 0.f, m1 = 0.f;
      float2 s1 = f2(0.f), s3 = f2(0.f);
      float amx = 0.f, dmx = 0.f;
      if (i < N) {
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
      sx = pow2_scale(warp_max(amx));
      sz = pow2_scale(2.f * warp_max(dmx));
      __syncwarp();   // every lane has its row in registers: Z' may now overwrite the slice
      if (i < N) {
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
      } else {
        // padding rows of Z' (the Gram's K rows j >= N) are zero
#pragma unroll
        for (int q = 0; q < 3; q++) {
          *reinterpret_cast<uint4*>(z_hi + i * 24 + 8 * q) = make_uint4(0, 0, 0, 0);
          *reinterpret_cast<uint4*>(z_lo + i * 24 + 8 * q) = make_uint4(0, 0, 0, 0);
        }
      }
      __syncwarp();

      // ---------------- a3: Gram G' = Z' Z'^T (= sz^2 G), K = 16 + 8
#pragma unroll
      for (int mt = 0; mt < MT; mt++)
#pragma unroll
        for (int nt = 0; nt < 2 * MT; nt++)
#pragma unroll
          for (int e = 0; e < 4; e++) g[mt][nt][e] = 0.f;
      {
        uint32_t ah[MT][4], al[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; mt++) {
          const int off = (16 * mt + (lane & 7) + 8 * (q8 & 1)) * 24 + 8 * (q8 >> 1);
          ldsm_x4(ah[mt], z_hi + off);
          ldsm_x4(al[mt], z_lo + off);
        }
#pragma unroll
        for (int np = 0; np < MT; np++) {
          uint32_t bh[4], bl[4];
          const int off = (16 * np + (lane & 7) + 8 * (q8 >> 1)) * 24 + 8 * (q8 & 1);
          ldsm_x4(bh, z_hi + off);
          ldsm_x4(bl, z_lo + off);
#pragma unroll
          for (int mt = 0; mt < MT; mt++) {
            mma16816(g[mt][2 * np], al[mt], bh[0], bh[1]);
            mma16816(g[mt][2 * np + 1], al[mt], bh[2], bh[3]);
          }
#pragma unroll
          for (int mt = 0; mt < MT; mt++) {
            mma16816(g[mt][2 * np], ah[mt], bl[0], bl[1]);
            mma16816(g[mt][2 * np + 1], ah[mt], bl[2], bl[3]);
          }
#pragma unroll
          for (int mt = 0; mt < MT; mt++) {
            mma16816(g[mt][2 * np], ah[mt], bh[0], bh[1]);
            mma16816(g[mt][2 * np + 1], ah[mt], bh[2], bh[3]);
          }
        }
        uint32_t th[MT][2], tl[MT][2];
#pragma unroll
        for (int mt = 0; mt < MT; mt++) {
          const int off = (16 * mt + (lane & 7) + 8 * (q8 & 1)) * 24 + 16;
          ldsm_x2(th[mt][0], th[mt][1], z_hi + off);
          ldsm_x2(tl[mt][0], tl[mt][1], z_lo + off);
        }
#pragma unroll
        for (int np = 0; np < MT; np++) {
          uint32_t bh[2], bl[2];
          const int off = (16 * np + 8 * (q8 & 1) + (lane & 7)) * 24 + 16;
          ldsm_x2(bh[0], bh[1], z_hi + off);
          ldsm_x2(bl[0], bl[1], z_lo + off);
#pragma unroll
          for (int mt = 0; mt < MT; mt++) {
            mma1688(g[mt][2 * np], tl[mt][0], tl[mt][1], bh[0]);
            mma1688(g[mt][2 * np + 1], tl[mt][0], tl[mt][1], bh[1]);
            mma1688(g[mt][2 * np], th[mt][0], th[mt][1], bl[0]);
            mma1688(g[mt][2 * np + 1], th[mt][0], th[mt][1], bl[1]);
            mma1688(g[mt][2 * np], th[mt][0], th[mt][1], bh[0]);
            mma1688(g[mt][2 * np + 1], th[mt][0], th[mt][1], bh[1]);
          }
        }
      }
      __syncwarp();   // Z' consumed: the slice now receives the attention tiles
    }
    // Def 5: sigma^2 = (1/(N S)) sum_n [nu2_n + S (mu_n - mubar)^2]
    const float mbar_ = warp_sum(i < N ? mu : 0.f) * a.inv_n;
    const float dv = i < N ? nu2 + (float)S * (mu - mbar_) * (mu - mbar_) : 0.f;
    const float inv_var = 1.0f / (warp_sum(dv) * a.inv_ns + kEpsTrend);

    // A slice word for (row i = 16 mt + 8 h + gq, cols j = 8 nt + 2 cq, +1), K chunk kc:
    // M chunk (warp*4 + nt) * 2048 + kc * 128 + gq * 16 + cq * 4 (MN-major core matrices)
    auto a_word = [&](int nt, int kc) -> uint32_t* {
      return reinterpret_cast<uint32_t*>(slice + nt * 2048 + kc * 128 + gq * 16 + cq * 4);
    };

    if (active) {
      // ---------------- a4+a5 trend (Def 7-8): exponent -(mu~_i - mu~_j)^2 - (k~_i - k~_j)^2,
      // row max 0 at j = i; A_t -> K columns 32..63 (hi), 96..127 (lo)
      {
        const float cm = sqrtf(inv_var * a.kt), ck = sqrtf(a.vtrend * inv_var * a.kt);
        const float mus = i < N ? mu * cm : 0.f, kas = i < N ? kap * ck : 0.f;
        float2 cmu[2 * MT], ckap[2 * MT];
#pragma unroll
        for (int nt = 0; nt < 2 * MT; nt++) {
          const int j = 8 * nt + 2 * cq;
          const float m0 = __shfl_sync(0xffffffffu, mus, j), m1v = __shfl_sync(0xffffffffu, mus, j + 1);
          cmu[nt] = make_float2(j < N ? -m0 : -INFINITY, j + 1 < N ? -m1v : -INFINITY);
          ckap[nt] = make_float2(-__shfl_sync(0xffffffffu, kas, j), -__shfl_sync(0xffffffffu, kas, j + 1));
        }
#pragma unroll
        for (int mt = 0; mt < MT; mt++)
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int ii = 16 * mt + 8 * h + gq;
            const float2 mui = f2(__shfl_sync(0xffffffffu, mus, ii));
            const float2 ki = f2(__shfl_sync(0xffffffffu, kas, ii));
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
            const float2 rs2 = f2(ii < N ? 1.f / sum : 0.f);
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
              *a_word(nt, 4 + 2 * mt + h) = hi;
              *a_word(nt, 12 + 2 * mt + h) = lo;
            }
          }
      }

      // ---------------- a5 seasonal (Def 6, 8): rho_ij = G'_ij inv_i inv_j / sz^2, row softmax;
      // A_s -> K columns 0..31 (hi), 64..95 (lo)
      {
        const float inv = i < N ? rsqrtf(nu2 + kEpsSeasonal) : 1.f;
        const float ks_z = a.ks / (sz * sz);
        float2 cinv[2 * MT], cmask[2 * MT];
#pragma unroll
        for (int nt = 0; nt < 2 * MT; nt++) {
          const int j = 8 * nt + 2 * cq;
          cinv[nt] = make_float2(__shfl_sync(0xffffffffu, inv, j), __shfl_sync(0xffffffffu, inv, j + 1));
          cmask[nt] = make_float2(j < N ? 0.f : -INFINITY, j + 1 < N ? 0.f : -INFINITY);
        }
#pragma unroll
        for (int mt = 0; mt < MT; mt++)
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int ii = 16 * mt + 8 * h + gq;
            const float rk = __shfl_sync(0xffffffffu, inv, ii) * ks_z;
            float2 u[2 * MT];
            float mx = -INFINITY;
#pragma unroll
            for (int nt = 0; nt < 2 * MT; nt++) {
              u[nt] = fma2(make_float2(g[mt][nt][2 * h], g[mt][nt][2 * h + 1]), cinv[nt], cmask[nt]);
              mx = fmaxf(mx, fmaxf(u[nt].x, u[nt].y));
            }
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const float2 rk2 = f2(rk), nb2 = f2(-mx * rk);
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
            const float2 rs2 = f2(ii < N ? 1.f / sum : 0.f);
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
              *a_word(nt, 2 * mt + h) = hi;
              *a_word(nt, 8 + 2 * mt + h) = lo;
            }
          }
      }
    }

    // ---------------- a6+a7 fold on tcgen05: Q'^T[(w, j)][m] = sum_i Acat^T[(w, j)][i] W'^T[i][m]
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // A tile -> async proxy
    tc_fence_before();
    group_bar(1, 128);
    tc_fence_after();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int ks = 0; ks < 4; ks++) {
        const uint64_t ah = smem_desc(a_base + ks * 256, 128, 2048);
        const uint64_t al = smem_desc(a_base + (8 + 2 * ks) * 128, 128, 2048);
        const uint64_t bh = smem_desc(w_base + ks * 256, 128, 2048);
        const uint64_t bl = smem_desc(w_base + (8 + 2 * ks) * 128, 128, 2048);
        tc_mma_f16(tmem_d, ah, bh, kIdesc, ks > 0 ? 1u : 0u);
        tc_mma_f16(tmem_d, ah, bl, kIdesc, 1u);
        tc_mma_f16(tmem_d, al, bh, kIdesc, 1u);
      }
      tc_commit(mbar);
    }
    mbar_wait_bounded(mbar, mphase);
    mphase ^= 1u;
    tc_fence_after();
    float qv[32];
    tmem_ld32(tmem_d + ((uint32_t)(32 * warp) << 16), qv);   // lane j: Q'[0..31][j]
    // the slice's A data is consumed: stage the next series into it (TMA) now
    const int64_t bn = b + 4;
    if (bn < b_end) issue_load(bn);

    if (active) {
      // ---------------- Q' -> fp16 hi/lo, staged [j][m] so ldmatrix.trans yields A fragments
      {
        uint32_t* qh = reinterpret_cast<uint32_t*>(qst + lane * kTcQRow);
        uint32_t* ql = reinterpret_cast<uint32_t*>(qst + 32 * kTcQRow + lane * kTcQRow);
#pragma unroll
        for (int q = 0; q < 4; q++) {
          uint4 vh, vl;
          uint32_t* ph = reinterpret_cast<uint32_t*>(&vh);
          uint32_t* pl = reinterpret_cast<uint32_t*>(&vl);
#pragma unroll
          for (int u = 0; u < 4; u++) split2(qv[8 * q + 2 * u], qv[8 * q + 2 * u + 1], ph[u], pl[u]);
          reinterpret_cast<uint4*>(qh)[q] = vh;
          reinterpret_cast<uint4*>(ql)[q] = vl;
        }
      }
      __syncwarp();

      // ---------------- a7 head Y' = Q' X' (= sw sx Y) on mma.sync; a8 store y = Y + b
      const float2 ys2 = f2(inv_sw / sx);
      float* yg = a.y + series * H;
#pragma unroll
      for (int mm = 0; mm < MMT; mm++) {
        if (16 * mm >= M) break;
        uint32_t qh[MT][4], ql[MT][4];
#pragma unroll
        for (int kj = 0; kj < MT; kj++) {
          const int off = (16 * kj + 8 * (q8 >> 1) + (lane & 7)) * kTcQRow + (16 * mm + 8 * (q8 & 1)) * 2;
          ldsm_x4_t(qh[kj], qst + off);
          ldsm_x4_t(ql[kj], qst + 32 * kTcQRow + off);
        }
        float ya[3][4];
#pragma unroll
        for (int nt = 0; nt < 3; nt++)
#pragma unroll
          for (int e = 0; e < 4; e++) ya[nt][e] = 0.f;
#pragma unroll
        for (int kj = 0; kj < MT; kj++) {
          uint32_t xh[4], xl[4], xh2[2], xl2[2];
          const int krow = 16 * kj + (lane & 7) + 8 * (q8 & 1);
          ldsm_x4_t(xh, x_hi + krow * 24 + 8 * (q8 >> 1));
          ldsm_x4_t(xl, x_lo + krow * 24 + 8 * (q8 >> 1));
          ldsm_x2_t(xh2[0], xh2[1], x_hi + krow * 24 + 16);
          ldsm_x2_t(xl2[0], xl2[1], x_lo + krow * 24 + 16);
          mma16816(ya[0], ql[kj], xh[0], xh[1]);
          mma16816(ya[1], ql[kj], xh[2], xh[3]);
          mma16816(ya[2], ql[kj], xh2[0], xh2[1]);
          mma16816(ya[0], qh[kj], xl[0], xl[1]);
          mma16816(ya[1], qh[kj], xl[2], xl[3]);
          mma16816(ya[2], qh[kj], xl2[0], xl2[1]);
          mma16816(ya[0], qh[kj], xh[0], xh[1]);
          mma16816(ya[1], qh[kj], xh[2], xh[3]);
          mma16816(ya[2], qh[kj], xh2[0], xh2[1]);
        }
#pragma unroll
        for (int nt = 0; nt < 3; nt++) {
          const int t = 8 * nt + 2 * cq;
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int m = 16 * mm + 8 * h + gq;
            const int hh = m * S + t;
            if (m < M && hh < H) {
              const float2 v = mul2(make_float2(ya[nt][2 * h], ya[nt][2 * h + 1]), ys2);
              if ((H & 1) == 0) {
                const float2 o = add2(v, *reinterpret_cast<const float2*>(bS + hh));
                asm volatile("st.global.cs.v2.f32 [%0], {%1,%2};" ::"l"(yg + hh), "f"(o.x),
                             "f"(o.y)
                             : "memory");
              } else {
                yg[hh] = v.x + bS[hh];
                if (hh + 1 < H) yg[hh + 1] = v.y + bS[hh + 1];
              }
            }
          }
        }
      }
    }
    __syncwarp();
  }
  cp_async_wait_all();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem_d, 32);
}

bool plan_tc_kernel(const FwdArgs& a, int max_smem_optin, TcPlan* p) {
  if (a.S != 24 || a.N <= 16 || a.N > 32 || a.M > 32) return false;
  p->mmt = a.M <= 16 ? 1 : 2;
  p->smem_bytes = (size_t)kTcOffBias + (size_t)a.H * 4;
  if (p->smem_bytes > (size_t)max_smem_optin) return false;
  p->wins_per_cta = 128;
  return true;
}

template <int MMT, bool DBG>
static cudaError_t launch_tc_t(const FwdArgs& a, const TcPlan& p, cudaStream_t st) {
  auto k = prnet_fwd_tc_kernel<MMT, DBG>;
  cudaError_t e =
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((a.B + p.wins_per_cta - 1) / p.wins_per_cta), (unsigned)a.C);
  k<<<grid, 128, p.smem_bytes, st>>>(a, p.wins_per_cta);
  return cudaGetLastError();
}

cudaError_t launch_tc_kernel(const FwdArgs& a, const TcPlan& p, cudaStream_t st) {
  const bool dbg = a.a_s_dbg != nullptr;
  if (p.mmt == 1) return dbg ? launch_tc_t<1, true>(a, p, st) : launch_tc_t<1, false>(a, p, st);
  return dbg ? launch_tc_t<2, true>(a, p, st) : launch_tc_t<2, false>(a, p, st);
}

}  // namespace prnet
