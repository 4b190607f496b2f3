// fwd_tcl.cu -- "tc_long": the PRNet pattern-attention forward for long lookbacks
// (32 < N <= 512 segments, S in {12, 24, 48, 96}, M <= 32; the long end of the BASELINE.json
// configs[4] stress sweep) on the 5th-gen tensor cores, flash-attention style.
//
// Same reading (SURVEY §8(c) Definition steps 1-11) and split-fp16 3-product
// arithmetic as every other variant.  One CTA of 16 warps owns one series at a
// time (the CTA walks a contiguous window range of one channel):
//
//  a1/a2  the series (N S floats) arrives by 1-D bulk copies into one of two staging buffers
//         (the next series is fetched while this one is processed); thread r computes the
//         descriptors of segment r and writes its Z' row (K-major, [hi t | lo t]) and its X'
//         row (MN-major B operand, [t][key]) as split fp16; sigma^2 and the X' scale are CTA
//         reductions;
//  a3     per (query tile of 128 rows, key tile of 64 rows): G = Z'_q Z'_k^T on tcgen05.mma
//         (SS, TMEM accumulator, 64 columns);
//  a4/a5  thread (row quarter w%4, column quarter w/4) reads 16 columns of its row of G
//         (tcgen05.ld), forms the seasonal exponentials 2^((rho_ij - f_i) ks) with the KNOWN row
//         bound f_i = nu_i / sqrt(nu_i^2 + eps_s) >= rho_ij (Cauchy-Schwarz; no online
//         rescaling) and the trend exponentials 2^(-(mu~_i - mu~_j)^2 - (k~_i - k~_j)^2) (row max
//         0 at j = i), accumulates row sums, and stores E as split fp16 into TMEM (two
//         buffers, so the next key tile's exponentials never wait for this tile's MMA);
//  a6     P_s += E_s X'_k, P_t += E_t X'_k on tcgen05.mma (TS: E from TMEM, X' from shared
//         memory), P in TMEM; the Gram of the next tile is issued as soon as G is read;
//  a7     per query tile, 4 warps fold the normalised patterns into the head (per-warp
//         mma.sync, W' fragments from the flash head pack, P^T by movmatrix), partial Y in
//         fixed-order shared-memory slots;
//  a8     y = Y / (sw sx) + b, coalesced stores by the whole CTA.
//
// TMEM (512 columns): G [0,64) | E buffer 0 [64,192) | E buffer 1 [192,320) | P_s, P_t
// [320, 320 + 2 SP); an E buffer = E_s hi, E_s lo, E_t hi, E_t lo (32 columns each: 64 keys
// packed two per column).  Every tcgen05.mma is issued by thread 0, so each commit covers all
// earlier MMAs: waiting for the Gram of tile k+2 also proves the P-MMA of tile k (the reader
// of the E buffer about to be rewritten) complete.
#include <cuda_fp16.h>

#include <cmath>

#include "tc_common.cuh"

// ablation switches for A/B builds (results invalid when non-zero): 1 no P-MMA, 2 no Gram MMA,
// 4 no exponentials, 8 no head
// the MMA thread's mbarrier waits carry a suspend-time hint (ns; 0 = plain polling).  A/B
// (profiles/README.md): 2000 ns 0.7-0.9 % faster at S <= 24 than polling, equal at S = 48
#ifndef PRNET_TCL_SLEEP_NS
#define PRNET_TCL_SLEEP_NS 2000
#endif
#ifndef PRNET_TCL_ABL
#define PRNET_TCL_ABL 0
#endif

namespace prnet {
using namespace tcq;

namespace {

// NWS = softmax warps: 16 (one CTA per SM, 512 TMEM columns: two E buffers and, when they fit,
// two G buffers) or 8 (two CTAs per SM, 256 columns each: one G, one E buffer, S <= 24; every
// softmax thread then covers 32 of a tile's 64 keys)
template <int S, int NWS = 16>
struct TclCfg {
  static_assert(S % 4 == 0 && S <= 96, "S");
  static_assert(NWS == 16 || NWS == 8, "NWS");
  static constexpr int SP = (S + 15) / 16 * 16;   // Gram K per product; P columns
  static constexpr int NCT = (S + 7) / 8;         // head n-tiles
  static constexpr int NQ = S / 4;
  static constexpr int PITCH = ((S / 4) & 1) ? 4 * S : 4 * S + 16;   // staging row bytes
  static constexpr bool ROWCOPY = PITCH != 4 * S;
  static constexpr int SBO = 32 * SP;             // Z' row block stride (8 rows x 2 SP halves)
  static constexpr int TB = NWS == 16 ? 512 : 256;   // TMEM columns of the CTA
  static constexpr int EB = NWS == 16 ? 2 : 1;        // E buffers (128 columns each)
  // P-MMA B operand: NM = 2 -> [X' hi | X' lo] as one N = 2 SP operand (the lo tile follows the
  // hi tile along N), so each E half is read once per K-step: D = [hh + lh | hl + ll] per
  // branch (P = the two halves summed); NM = 1 -> N = SP, three products hh, hl, lh
  static constexpr int NM = 64 + 128 * EB + 4 * SP <= TB ? 2 : 1;
  static constexpr int PW = NM * SP;                // P columns per branch
  // TMEM columns: G buffers (64 each; two when they fit), E buffers, P_s | P_t
  static constexpr int GB = 128 + 128 * EB + 2 * PW <= TB ? 2 : 1;
  static constexpr uint32_t TG = 0, TE0 = 64 * GB, TE1 = TE0 + 128, TP = TE0 + 128 * EB;
  static_assert(TP + 2 * PW <= TB, "TMEM");
  static constexpr int NWC = NWS / 4;               // column groups of the softmax warps
  static constexpr int CPT = 64 / NWC;              // keys per softmax thread and tile
  static constexpr int NT = 32 * (NWS + 1);         // threads (+ the MMA warp)
  static constexpr int RPT = (512 + NT - 1) / NT;   // descriptor rows per thread (N <= 512)
  static constexpr int SB = NWS == 16 ? 2 : 1;      // staging buffers
};

__device__ __forceinline__ void sts128(unsigned char* p, uint4 v) {
  *reinterpret_cast<uint4*>(p) = v;
}
__device__ __forceinline__ void bulk_copy_tx(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
template <int S>
__device__ __forceinline__ constexpr float ttl(int t) {
  return (float)t - 0.5f * (float)(S - 1);
}
__device__ __forceinline__ void tld_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : PRNET_TLD_R8(r, 0), PRNET_TLD_R8(r, 8)
      : "r"(taddr));
}
__device__ __forceinline__ void tst_x8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}
// 16x256b.x1: thread t <- lanes base + t/4 and base + 8 + t/4, columns 2(t%4), 2(t%4)+1
__device__ __forceinline__ void tld16_x1(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
// A fragment (16 x 16, rows r0.., cols c0..) of a row-major global fp16 matrix
__device__ __forceinline__ void ldg_afrag16(const __half* base, int ld, int r0, int c0, int lane,
                                            uint32_t (&f)[4]) {
  const int g = lane >> 2, c = lane & 3;
  const __half* p = base + (size_t)(r0 + g) * ld + c0 + 2 * c;
  f[0] = __ldg(reinterpret_cast<const unsigned int*>(p));
  f[1] = __ldg(reinterpret_cast<const unsigned int*>(p + 8 * ld));
  f[2] = __ldg(reinterpret_cast<const unsigned int*>(p + 8));
  f[3] = __ldg(reinterpret_cast<const unsigned int*>(p + 8 * ld + 8));
}

// The exponentials of one thread's 16 key columns (a4/a5): seasonal 2^(rho ks - f_i ks), trend
// 2^(-(mu~_i - mu~_j)^2 - (k~_i - k~_j)^2), split fp16 hi/lo for the TMEM store, row sums added
// to ls / lt.  MASK: columns j >= nvalid get 0 (the last key tile only).
template <bool MASK>
__device__ __forceinline__ void tcl_exps(const uint32_t (&g)[16], float ks, float fk, float mi,
                                         float ki, const float* mt, const float* kt, int nvalid,
                                         uint32_t (&eh)[8], uint32_t (&el)[8], uint32_t (&th)[8],
                                         uint32_t (&tlo)[8], float& ls, float& lt) {
  const float2 ks2 = f2(ks), nf2 = f2(-fk);
  float2 sa2 = f2(0.f), sb2 = f2(0.f);
#pragma unroll
  for (int j = 0; j < 16; j += 2) {
    const float2 arg = fma2(make_float2(__uint_as_float(g[j]), __uint_as_float(g[j + 1])), ks2, nf2);
    float e0 = fast_ex2(arg.x), e1 = fast_ex2(arg.y);
    if (MASK) {
      e0 = j < nvalid ? e0 : 0.f;
      e1 = j + 1 < nvalid ? e1 : 0.f;
    }
    if (j & 2) sb2 = add2(sb2, make_float2(e0, e1));
    else sa2 = add2(sa2, make_float2(e0, e1));
    split2(make_float2(e0, e1), eh[j / 2], el[j / 2]);
  }
  const float2 s2 = add2(sa2, sb2);
  ls += s2.x + s2.y;
  const float2 mi2 = f2(mi), ki2 = f2(ki);
  const float4* cm4 = reinterpret_cast<const float4*>(mt);
  const float4* ck4 = reinterpret_cast<const float4*>(kt);
  float2 ta2 = f2(0.f), tb2 = f2(0.f);
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const float4 mj = cm4[q], kj = ck4[q];
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int j = 4 * q + 2 * h;
      const float2 dm = add2(mi2, h ? make_float2(-mj.z, -mj.w) : make_float2(-mj.x, -mj.y));
      const float2 dk = add2(ki2, h ? make_float2(-kj.z, -kj.w) : make_float2(-kj.x, -kj.y));
      const float2 ex = fma2(make_float2(-dk.x, -dk.y), dk, mul2(make_float2(-dm.x, -dm.y), dm));
      float e0 = fast_ex2(ex.x), e1 = fast_ex2(ex.y);
      if (MASK) {
        e0 = j < nvalid ? e0 : 0.f;
        e1 = j + 1 < nvalid ? e1 : 0.f;
      }
      if (h) tb2 = add2(tb2, make_float2(e0, e1));
      else ta2 = add2(ta2, make_float2(e0, e1));
      split2(make_float2(e0, e1), th[j / 2], tlo[j / 2]);
    }
  }
  const float2 t2 = add2(ta2, tb2);
  lt += t2.x + t2.y;
}

}  // namespace

template <int S, int MT, int NWS>
__global__ void __launch_bounds__(32 * (NWS + 1), NWS == 16 ? 1 : 2) prnet_fwd_tcl_kernel(
    FwdArgs a, TclLayout ly, int ctas_per_channel) {
  using K = TclCfg<S, NWS>;
  extern __shared__ __align__(1024) unsigned char smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const bool mma_warp = warp == NWS;           // the last warp issues every tcgen05.mma (lane 0)
  const int wq = warp & 3, wc = (warp >> 2) % K::NWC;   // row quarter (TMEM lanes), column group
  const int c = blockIdx.y;
  const int cw = a.head_per_channel ? c : 0;
  const int N = a.N, M = a.M, H = a.H, C = a.C;
  const int NQT = ly.nqt, NKT = ly.nkt, NK = 64 * NKT;

  unsigned char* zt = smem + ly.off_z;
  unsigned char* xhi = smem + ly.off_x;
  unsigned char* xlo = xhi + 2 * K::SP * NK;
  unsigned char* const stg0 = smem + ly.off_stage;
  float* fks = reinterpret_cast<float*>(smem + ly.off_vec);    // [Rpad] f_i ks (seasonal shift)
  float* mtv = fks + ly.rpad;                                  // [Rpad] mu~
  float* ktv = mtv + ly.rpad;                                  // [Rpad] kappa~
  float* lpart = ktv + ly.rpad;                                // [2][NWC][128] row-sum partials
  float* red = lpart + 2 * 4 * 128;                            // [17][3] reduction scratch, [63] m0
  float* yslot = reinterpret_cast<float*>(smem + ly.off_y);    // [2 branch][4 wq][16 MT][8 NCT]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ly.off_bar);
  uint64_t* gfree = bars + 12;   // [GB] 16 softmax warps have read G buffer b (per-buffer
                                 // barriers: a completion two tiles ahead needs the next Gram)
  uint64_t* gfull = bars + 10;   // [GB] Gram into G buffer b committed (tcgen05.commit)
  uint64_t* efull = bars + 2;    // [2] 16 softmax warps have stored E buffer b
  uint64_t* efree = bars + 4;    // [2] P-MMA reading E buffer b committed
  uint64_t* pfull = bars + 6;    // last P-MMA of a query tile committed
  uint64_t* pfree = bars + 7;    // 16 softmax warps have read P (the head)
  uint64_t* xbar = bars + 8;     // [2] staging buffers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + ly.off_bar + 128);
  constexpr int YW = 16 * MT * 8 * K::NCT;                     // floats per Y slot

  if (tid == 0) {
    mbar_init(gfull, 1);
    mbar_init(gfull + 1, 1);
    mbar_init(gfree, NWS);
    mbar_init(gfree + 1, NWS);
    mbar_init(efull, NWS);
    mbar_init(efull + 1, NWS);
    mbar_init(efree, 1);
    mbar_init(efree + 1, 1);
    mbar_init(pfull, 1);
    mbar_init(pfree, NWS);
    mbar_init(xbar, 1);
    mbar_init(xbar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int k = tid; k < 8 * YW; k += blockDim.x) yslot[k] = 0.f;
  if (warp == 0) tmem_alloc(tmem_slot, K::TB);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem0 = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const uint32_t tl = tmem0 + ((uint32_t)(32 * wq) << 16);   // this warp's lanes
  const uint32_t z_s = smem_u32(zt), xhi_s = smem_u32(xhi), xlo_s = smem_u32(xlo);
  const float inv_sw = __ldg(a.wpack_flash_inv_sw + cw);
  const int npf = (N + 15) & ~15;                 // the flash head pack's K padding
  const int ldw = 2 * npf;
  const __half* whi = reinterpret_cast<const __half*>(a.wpack_flash) +
                      (size_t)cw * (ly.wpack_bytes / 2);
  const __half* wlo = whi + (M <= 16 ? 16 : (M <= 32 ? 32 : 64)) * ldw;

  const int64_t b0 = a.B * blockIdx.x / ctas_per_channel;
  const int64_t b1 = a.B * (blockIdx.x + 1) / ctas_per_channel;
  const int NS = N * S;
  const bool bulk = a.x_vec;
  auto xptr = [&](int64_t b) { return a.x + b * a.xsb + c * a.xsc + a.r; };
  // series -> staging buffer (thread 0 arms the barrier; row copies by warp 0's lanes, or one
  // span copy; unaligned windows: 4-byte cp.async by the softmax threads)
  auto issue_load = [&](int64_t b, int buf) {
    const float* xg = xptr(b);
    unsigned char* st = stg0 + (buf ? ly.stage_bytes : 0);
    if (bulk) {
      if (warp == 0) {
        if constexpr (K::ROWCOPY) {
          if (lane == 0) mbar_expect(xbar + buf, (uint32_t)NS * 4u);
          __syncwarp();
          for (int n = lane; n < N; n += 32) bulk_copy_tx(st + n * K::PITCH, xg + n * S, 4u * S, xbar + buf);
        } else {
          if (lane == 0) bulk_load(st, xg, (uint32_t)NS * 4u, xbar + buf);
        }
      }
    } else if (!mma_warp) {
      for (int k = tid; k < NS; k += 32 * NWS) {
        const int n = k / S, t = k - n * S;
        cp_async4(st + n * K::PITCH + 4 * t, xg + k);
      }
      cp_async_commit();
    }
  };

  // tile counter (query tile x key tile, over every series of the CTA): mbarrier parities
  uint32_t tile = 0, qcount = 0, phX = 0;
  if (b0 < b1) {
    fence_proxy_async();
    issue_load(b0, 0);
  }
  int buf = 0;
  for (int64_t b = b0; b < b1; b++, buf = K::SB == 2 ? buf ^ 1 : 0) {
    // ---------------- a1+a2: wait for this series (two buffers: prefetch the next one now)
    if (bulk) {
      mbar_wait_bounded(xbar + buf, (phX >> buf) & 1u);
      phX ^= 1u << buf;
    } else {
      cp_async_wait_all();
      __syncthreads();
    }
    if (K::SB == 2 && b + 1 < b1) {
      fence_proxy_async();
      issue_load(b + 1, buf ^ 1);
    }
    const float4* st4 = reinterpret_cast<const float4*>(stg0 + (buf ? ly.stage_bytes : 0));
    // segment rows r = tid + k NT (N <= 512): descriptors, Z' rows
    float mu_[K::RPT], kap_[K::RPT], nu2_[K::RPT];
    float s_a = 0.f, s_b = 0.f, bnd = 0.f, mu00 = 0.f;
#pragma unroll
    for (int rk = 0; rk < K::RPT; rk++) {
    const int r = tid + rk * K::NT;
    const bool rv = r < N;
    const float4* xr4 = st4 + (rv ? r : 0) * (K::PITCH / 16);
    float mu = 0.f, kap = 0.f, nu2 = 0.f, x0 = 0.f, m1 = 0.f;
    if (rv) {
      x0 = reinterpret_cast<const float*>(xr4)[0];
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
      m1 = (s1.x + s1.y) * a.inv_s;
      mu = x0 + m1;
      kap = (s3.x + s3.y) * a.inv_v;
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
      nu2 = q2.x + q2.y;
    }
    // Z' row r = z / sqrt(nu2 + eps_s) (rows N..Rpad-1 zero)
    if (r < ly.rpad) {
      const float zsc = rv ? rsqrtf(nu2 + kEpsSeasonal) : 0.f;
      const float2 zs2 = f2(zsc), nx0 = f2(-x0), nm1 = f2(-m1);
      unsigned char* zr = zt + (r >> 3) * K::SBO + (r & 7) * 16;
#pragma unroll
      for (int ch = 0; ch < K::SP / 8; ch++) {
        uint4 hv = make_uint4(0u, 0u, 0u, 0u), lv = make_uint4(0u, 0u, 0u, 0u);
        if (8 * ch < S) {
          const float4 v0 = xr4[2 * ch];
          split2(mul2(add2(add2(make_float2(v0.x, v0.y), nx0), nm1), zs2), hv.x, lv.x);
          split2(mul2(add2(add2(make_float2(v0.z, v0.w), nx0), nm1), zs2), hv.y, lv.y);
          if (8 * ch + 4 < S) {
            const float4 v1 = xr4[2 * ch + 1];
            split2(mul2(add2(add2(make_float2(v1.x, v1.y), nx0), nm1), zs2), hv.z, lv.z);
            split2(mul2(add2(add2(make_float2(v1.z, v1.w), nx0), nm1), zs2), hv.w, lv.w);
          }
        }
        if (!rv) { hv = make_uint4(0u, 0u, 0u, 0u); lv = hv; }
        sts128(zr + ch * 128, hv);
        sts128(zr + (K::SP / 8 + ch) * 128, lv);
      }
    }
    mu_[rk] = mu;
    kap_[rk] = kap;
    nu2_[rk] = nu2;
    if (rk == 0) mu00 = mu;
    }
    // CTA reductions: sum (mu - m0), sum [S (mu - m0)^2 + nu2] (sigma^2, Def 5, about the
    // reference m0 = mu_0) and max (|mu| + |z|) (the X' scale); m0 from thread 0 via smem
    if (tid == 0) red[63] = mu00;
    __syncthreads();
    const float m0 = red[63];
#pragma unroll
    for (int rk = 0; rk < K::RPT; rk++) {
      const bool rv = tid + rk * K::NT < N;
      const float dd = rv ? mu_[rk] - m0 : 0.f;
      s_a += dd;
      s_b += rv ? fmaf((float)S * dd, dd, nu2_[rk]) : 0.f;
      bnd = fmaxf(bnd, rv ? fabsf(mu_[rk]) + fast_sqrt(nu2_[rk]) : 0.f);
    }
    {
      s_a = warp_sum(s_a);
      s_b = warp_sum(s_b);
      const float mx = warp_max_nonneg(bnd);
      if (lane == 0) {
        red[3 * warp] = s_a;
        red[3 * warp + 1] = s_b;
        red[3 * warp + 2] = mx;
      }
    }
    __syncthreads();
    float sa = 0.f, sb = 0.f, mxa = 0.f;
#pragma unroll
    for (int w = 0; w < NWS + 1; w++) {
      sa += red[3 * w];
      sb += red[3 * w + 1];
      mxa = fmaxf(mxa, red[3 * w + 2]);
    }
    const float var = fmaf(-(float)S * sa, sa * a.inv_n, sb) * a.inv_ns;
    // series-level factors once (MUFU reciprocal / square root, <= ~1 ulp), not per row
    const float inv_var = fast_rcp(var + kEpsTrend);
    const float tsc = fast_sqrt(inv_var * a.kt), tsk = tsc * fast_sqrt(a.vtrend);
    const float sx = pow2_scale(mxa);
#pragma unroll
    for (int rk = 0; rk < K::RPT; rk++) {
    const int r = tid + rk * K::NT;
    const bool rv = r < N;
    const float4* xr4 = st4 + (rv ? r : 0) * (K::PITCH / 16);
    const float mu = mu_[rk], kap = kap_[rk], nu2 = nu2_[rk];
    // X' row r (MN-major B of the P-MMA: element (t, key r) at (t/8) 16 NK + (r/8) 128 +
    // (r%8) 16 + (t%8) 2), rows N..NK-1 zero; the per-row vectors
    if (r < NK) {
      const float2 xs2 = f2(rv ? sx : 0.f);
#pragma unroll
      for (int ch = 0; ch < K::SP / 8; ch++) {
        uint4 hv = make_uint4(0u, 0u, 0u, 0u), lv = make_uint4(0u, 0u, 0u, 0u);
        if (8 * ch < S) {
          const float4 v0 = xr4[2 * ch];
          split2(mul2(make_float2(v0.x, v0.y), xs2), hv.x, lv.x);
          split2(mul2(make_float2(v0.z, v0.w), xs2), hv.y, lv.y);
          if (8 * ch + 4 < S) {
            const float4 v1 = xr4[2 * ch + 1];
            split2(mul2(make_float2(v1.x, v1.y), xs2), hv.z, lv.z);
            split2(mul2(make_float2(v1.z, v1.w), xs2), hv.w, lv.w);
          }
        }
        const int o = ch * 16 * NK + (r >> 3) * 128 + (r & 7) * 16;
        sts128(xhi + o, hv);
        sts128(xlo + o, lv);
      }
    }
    if (r < ly.rpad) {
      // f_i = nu_i / sqrt(nu_i^2 + eps_s) >= rho_ij: the seasonal shift (rows >= N: 0)
      fks[r] = rv ? fast_sqrt(nu2) * rsqrtf(nu2 + kEpsSeasonal) * a.ks : 0.f;
      mtv[r] = rv ? mu * tsc : 0.f;
      ktv[r] = rv ? kap * tsk : 0.f;
    }
    }
    if (K::SB == 1) {   // the staging buffer is read: fetch the next series now
      __syncthreads();
      if (b + 1 < b1) {
        fence_proxy_async();
        issue_load(b + 1, 0);
      }
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    const int ntiles = NQT * NKT;
    if (mma_warp) {
      // ---------------- the MMA warp: Gram of tile t+1 as soon as G(t) is read, P-MMA of tile t
      // as soon as E(t) is stored; commits drive the softmax warps
      if (lane == 0) {
        const uint32_t sbo_x = 16u * (uint32_t)NK;
        // the MMA thread's waits: with PRNET_TCL_SLEEP_NS a suspend-time hint (the thread sleeps
        // until the phase completes instead of re-polling, leaving issue slots to the softmax
        // warps of the SM)
        auto mma_wait = [](uint64_t* bar, uint32_t parity) {
#if PRNET_TCL_SLEEP_NS
          mbar_wait_sleep(bar, parity, PRNET_TCL_SLEEP_NS);
#else
          mbar_wait_bounded(bar, parity);
#endif
        };
        auto issue_gram = [&](int t) {   // series tile t -> G buffer (tile + t) % GB
          const int qt = t / NKT, kt = t - qt * NKT;
          const uint32_t gb = K::GB == 2 ? ((tile + (uint32_t)t) & 1u) : 0u;
          const uint32_t dg = tmem0 + K::TG + 64u * gb;
          const uint32_t za = z_s + 16 * qt * K::SBO, zb = z_s + 8 * kt * K::SBO;
          constexpr uint32_t LO = (K::SP / 8) * 128;
          constexpr uint32_t id = idesc_f16(128, 64, false, false);
#pragma unroll
          for (int k = 0; k < ((PRNET_TCL_ABL & 2) ? 0 : K::SP / 16); k++) {
            const uint32_t o = k * 256;
            umma(dg, sdesc(za + o, 128, K::SBO), sdesc(zb + o, 128, K::SBO), id, k > 0);
            umma(dg, sdesc(za + o, 128, K::SBO), sdesc(zb + LO + o, 128, K::SBO), id, true);
            umma(dg, sdesc(za + LO + o, 128, K::SBO), sdesc(zb + o, 128, K::SBO), id, true);
          }
          umma_commit(gfull + gb);
        };
        issue_gram(0);
        if (K::GB == 2 && ntiles > 1) issue_gram(1);
        for (int t = 0; t < ntiles; t++) {
          const uint32_t tg = tile + (uint32_t)t;   // global tile index
          const int qt = t / NKT, kt = t - qt * NKT;
          if (t + K::GB < ntiles) {   // G buffer of tile t is read: the Gram of tile t + GB
            if (K::GB == 2) mma_wait(gfree + (tg & 1u), (tg >> 1) & 1u);
            else mma_wait(gfree, tg & 1u);
            tc_fence_after();
            issue_gram(t + K::GB);
          }
          if (kt == 0 && qcount + qt > 0) {   // the previous query tile's head has read P
            mma_wait(pfree, (qcount + qt - 1) & 1u);
            tc_fence_after();
          }
          const uint32_t eb = K::EB == 2 ? (tg & 1u) : 0u;
          mma_wait(efull + eb, K::EB == 2 ? ((tg >> 1) & 1u) : (tg & 1u));
          tc_fence_after();
          const uint32_t te = tmem0 + (eb ? K::TE1 : K::TE0);
          constexpr uint32_t id = idesc_f16(128, K::PW, false, true);
          // branches interleaved (consecutive MMAs accumulate into different D)
#pragma unroll
          for (int ks = 0; ks < ((PRNET_TCL_ABL & 1) ? 0 : 4); ks++) {
            const uint32_t ob = (uint32_t)(1024 * kt + 256 * ks);
            const uint64_t bh = sdesc(xhi_s + ob, 128, sbo_x), bl = sdesc(xlo_s + ob, 128, sbo_x);
            const bool acc = kt > 0 || ks > 0;
            const uint32_t d0 = tmem0 + K::TP, d1 = d0 + (uint32_t)K::PW;
            const uint32_t ah0 = te + 8u * ks, ah1 = ah0 + 64u;   // E_s hi, E_t hi
            if constexpr (K::NM == 2) {
              umma_ts(d0, ah0, bh, id, acc);
              umma_ts(d1, ah1, bh, id, acc);
              umma_ts(d0, ah0 + 32u, bh, id, true);
              umma_ts(d1, ah1 + 32u, bh, id, true);
            } else {
              umma_ts(d0, ah0, bh, id, acc);
              umma_ts(d1, ah1, bh, id, acc);
              umma_ts(d0, ah0, bl, id, true);
              umma_ts(d1, ah1, bl, id, true);
              umma_ts(d0, ah0 + 32u, bh, id, true);
              umma_ts(d1, ah1 + 32u, bh, id, true);
            }
          }
          umma_commit(efree + eb);
          if (kt + 1 == NKT) umma_commit(pfull);
        }
      }
      __syncwarp();
    } else {
      // ---------------- a3..a6 softmax warps over (query tile, key tile)
      for (int qt = 0; qt < NQT; qt++) {
        const int row = 128 * qt + 32 * wq + lane;   // this thread's query row
        const bool warp_rows = 128 * qt + 32 * wq < N;   // warp-uniform: any valid row
        const float fk = fks[row], mi = mtv[row], ki = ktv[row];
        float ls = 0.f, lt = 0.f;
        for (int kt = 0; kt < NKT; kt++) {
          const uint32_t tg = tile + (uint32_t)(qt * NKT + kt);
          const uint32_t eb = K::EB == 2 ? (tg & 1u) : 0u;
          const uint32_t te = tmem0 + (eb ? K::TE1 : K::TE0);
          const uint32_t gb = K::GB == 2 ? (tg & 1u) : 0u;
          mbar_wait_bounded(gfull + gb, K::GB == 2 ? ((tg >> 1) & 1u) : (tg & 1u));
          tc_fence_after();
          constexpr int NCH = K::CPT / 16;          // 16-key chunks of this thread
          uint32_t g[NCH][16];
#pragma unroll
          for (int h = 0; h < NCH; h++)
            tld_x16(tl + K::TG + 64u * gb + 16u * (uint32_t)(wc * NCH + h), g[h]);
          tld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(gfree + gb);
#pragma unroll
          for (int h = 0; h < NCH; h++) {
            const int cidx = wc * NCH + h;              // 16-key chunk of the tile
            const int j0 = 64 * kt + 16 * cidx;         // its first key
            uint32_t eh[8], el[8], th[8], tlo[8];
            // key columns past N (the last key tile) and rows past N (warp_rows false: no valid
            // key) take the separately compiled masked body, which writes zeros (no separate
            // zero-fill branch; measured neutral on B200, 25.03 vs 25.07 ms at stress L5760/S12)
            const int nv = warp_rows ? N - j0 : 0;
            if (nv >= 16)
              tcl_exps<false>(g[h], a.ks, fk, mi, ki, mtv + j0, ktv + j0, nv, eh, el, th, tlo, ls, lt);
            else
              tcl_exps<true>(g[h], a.ks, fk, mi, ki, mtv + j0, ktv + j0, nv, eh, el, th, tlo, ls, lt);
            if (h == 0) {
              // the E buffer is free once the P-MMA that last read it committed (two buffers:
              // tile tg - 2, one buffer: tile tg - 1)
              if (K::EB == 2 && tg >= 2) {
                mbar_wait_bounded(efree + eb, ((tg >> 1) - 1) & 1u);
                tc_fence_after();
              } else if (K::EB == 1 && tg >= 1) {
                mbar_wait_bounded(efree, (tg - 1) & 1u);
                tc_fence_after();
              }
            }
            // E into TMEM buffer eb: [0,32) E_s hi, [32,64) E_s lo, [64,96) E_t hi, [96,128)
            // E_t lo (a 16-key chunk = 8 packed columns at 8 cidx)
            tst_x8(tl + (te - tmem0) + 8u * cidx, eh);
            tst_x8(tl + (te - tmem0) + 32u + 8u * cidx, el);
            tst_x8(tl + (te - tmem0) + 64u + 8u * cidx, th);
            tst_x8(tl + (te - tmem0) + 96u + 8u * cidx, tlo);
          }
          tst_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(efull + eb);
        }
        // ---------------- a7: row sums -> 1/l; the head over this query tile's rows
        lpart[wc * 128 + 32 * wq + lane] = ls;
        lpart[K::NWC * 128 + wc * 128 + 32 * wq + lane] = lt;
        named_bar(1, 32 * NWS);
        mbar_wait_bounded(pfull, (qcount + qt) & 1u);
        tc_fence_after();
        if (warp_rows && !(PRNET_TCL_ABL & 8)) {
          const int g = lane >> 2;
          // 1 / l of this lane's fragment rows (branch, k-step, row half) by the MUFU reciprocal
          // (<= 1 ulp, as the other kernels' softmax); for MT <= 2 once per query tile rather than
          // per work item (measured: S = 96 10.58 -> 9.72 ms; with four head m-tiles, M > 32, the
          // hoisted copies cost registers, L5760/S12/H720 46.2 vs 47.0 ms, so MT = 4 recomputes)
          auto inv_l = [&](int br, int kb, int v) {
            const int rr = 32 * wq + 16 * kb + g + 8 * v;
            const float* lp = lpart + K::NWC * 128 * br + rr;
            float l_ = lp[0];
#pragma unroll
            for (int cg = 1; cg < K::NWC; cg++) l_ += lp[cg * 128];
            return 128 * qt + rr < N ? fast_rcp(l_) : 0.f;
          };
          float ilv[2][2][2];
          if constexpr (MT <= 2) {
#pragma unroll
            for (int br = 0; br < 2; br++)
#pragma unroll
              for (int kb = 0; kb < 2; kb++)
#pragma unroll
                for (int v = 0; v < 2; v++) ilv[br][kb][v] = inv_l(br, kb, v);
          }
          // work items (branch, n-tile) of this row quarter, split over the column quarters
          for (int it = wc; it < 2 * K::NCT; it += K::NWC) {
            const int br = it / K::NCT, nt = it - br * K::NCT;
            float acc[MT][4];
#pragma unroll
            for (int mt = 0; mt < MT; mt++)
#pragma unroll
              for (int e = 0; e < 4; e++) acc[mt][e] = 0.f;
#pragma unroll
            for (int kb = 0; kb < 2; kb++) {
              const int i0 = 128 * qt + 32 * wq + 16 * kb;   // K rows of this step
              if (i0 >= npf) break;
              float il[2];
              if constexpr (MT <= 2) {
                il[0] = br ? ilv[1][kb][0] : ilv[0][kb][0];
                il[1] = br ? ilv[1][kb][1] : ilv[0][kb][1];
              } else {
                il[0] = inv_l(br, kb, 0);
                il[1] = inv_l(br, kb, 1);
              }
              uint32_t pr[4];
              const uint32_t pa = tmem0 + ((uint32_t)(32 * wq + 16 * kb) << 16) + K::TP +
                                  (uint32_t)(br * K::PW + 8 * nt);
              tld16_x1(pa, pr);
              uint32_t pr2[4];
              if constexpr (K::NM == 2) tld16_x1(pa + (uint32_t)K::SP, pr2);
              uint32_t ah[MT][4], al[MT][4];
#pragma unroll
              for (int mt = 0; mt < MT; mt++) {
                ldg_afrag16(whi, ldw, 16 * mt, (br ? npf : 0) + i0, lane, ah[mt]);
                ldg_afrag16(wlo, ldw, 16 * mt, (br ? npf : 0) + i0, lane, al[mt]);
              }
              tld_wait();
              if constexpr (K::NM == 2) {   // P = [hh + lh] + [hl + ll]
#pragma unroll
                for (int e = 0; e < 4; e++)
                  pr[e] = __float_as_uint(__uint_as_float(pr[e]) + __uint_as_float(pr2[e]));
              }
              uint32_t h0, l0, h1, l1;
              split2(make_float2(__uint_as_float(pr[0]) * il[0], __uint_as_float(pr[1]) * il[0]), h0, l0);
              split2(make_float2(__uint_as_float(pr[2]) * il[1], __uint_as_float(pr[3]) * il[1]), h1, l1);
              const uint32_t bh0 = movm_t(h0), bh1 = movm_t(h1), bl0 = movm_t(l0), bl1 = movm_t(l1);
#pragma unroll
              for (int mt = 0; mt < MT; mt++) {
                mma16816_nv(acc[mt], al[mt], bh0, bh1);
                mma16816_nv(acc[mt], ah[mt], bl0, bl1);
                mma16816_nv(acc[mt], ah[mt], bh0, bh1);
              }
            }
            // fixed-order partial sums: slot (branch, row quarter) over the query tiles
            float* ys = yslot + (br * 4 + wq) * YW;
#pragma unroll
            for (int mt = 0; mt < MT; mt++)
#pragma unroll
              for (int e = 0; e < 4; e++) {
                const int m = 16 * mt + g + 8 * (e >> 1), t = 8 * nt + 2 * (lane & 3) + (e & 1);
                ys[m * (8 * K::NCT) + t] += acc[mt][e];
              }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(pfree);
        named_bar(1, 32 * NWS);   // lpart is rewritten by the next query tile
      }
    }
    tile += (uint32_t)ntiles;
    qcount += (uint32_t)NQT;
    __syncthreads();
    // ---------------- a8: y = (sum of the slots) / (sw sx) + b, coalesced over h
    {
      const float ysc = inv_sw / sx;
      float* yg = a.y + (b * C + c) * (int64_t)H;
      const float* bg = a.bias + (int64_t)cw * H;
      for (int h = tid; h < H; h += blockDim.x) {
        const int m = h / S, t = h - m * S;
        const int o = m * (8 * K::NCT) + t;
        float yv = 0.f;
#pragma unroll
        for (int k = 0; k < 8; k++) yv += yslot[k * YW + o];
        yg[h] = fmaf(yv, ysc, __ldg(bg + h));
      }
    }
    __syncthreads();
    for (int k = tid; k < 8 * YW; k += blockDim.x) yslot[k] = 0.f;
    // (the next series' Z' / X' writes follow the last P-MMA, whose completion was waited)
  }
  cp_async_wait_all();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem0, K::TB);
}

bool tcl_supported_s(int S) { return S == 12 || S == 24 || S == 48 || S == 96; }

bool plan_tcl_kernel(const FwdArgs& a, int max_smem_optin, int sm_count, TclPlan* p) {
  if (!tcl_supported_s(a.S) || a.N <= 32 || a.N > 512 || a.M > 64) return false;
  const int S = a.S, SP = (S + 15) / 16 * 16, NCT = (S + 7) / 8;
  const int pitch = ((S / 4) & 1) ? 4 * S : 4 * S + 16;
  TclLayout& ly = p->ly;
  ly.nqt = (a.N + 127) / 128;
  ly.nkt = (a.N + 63) / 64;
  ly.rpad = 128 * ly.nqt;
  const int NK = 64 * ly.nkt;
  const int MT = a.M <= 16 ? 1 : (a.M <= 32 ? 2 : 4);
  p->mt = MT;
  int off = 0;
  ly.off_z = off;
  off += ly.rpad * 4 * SP;                  // Z' [Rpad][hi SP | lo SP] halves
  ly.off_x = off;
  off += 4 * SP * NK;                       // X' hi | lo, [SP/8][NK/8] core matrices each
  ly.stage_bytes = (a.N * pitch + 127) & ~127;
  // two CTAs per SM (8 softmax warps, 256 TMEM columns, one staging buffer) when the S <= 24
  // instantiation's shared memory fits half the SM; else one CTA of 16 softmax warps
  const bool narrow = S <= 24;
  int off1 = off + ly.stage_bytes;
  const int vec = (3 * ly.rpad + 2 * 4 * 128 + 64) * 4;
  const int ybytes = 8 * 16 * MT * 8 * NCT * 4;
  const int tail = ((off1 + vec + 127) & ~127) - off1 + ybytes + 256;
  p->nws = (narrow && (size_t)(off1 + tail) <= (size_t)max_smem_optin / 2 - 1024) ? 8 : 16;
  ly.off_stage = off;
  off += (p->nws == 16 ? 2 : 1) * ly.stage_bytes;
  ly.off_vec = off;
  off += vec;
  off = (off + 127) & ~127;
  ly.off_y = off;
  off += ybytes;
  ly.off_bar = off;
  off += 256;
  ly.wpack_bytes = flash_wpack_bytes(a.N, a.M);
  p->smem_bytes = (size_t)off;
  if (p->smem_bytes > (size_t)max_smem_optin) return false;
  // channels x k CTAs, k against wave quantisation (1 or 2 CTAs per SM)
  const int64_t sms = (sm_count > 0 ? sm_count : 148) * (p->nws == 8 ? 2 : 1);
  int64_t best_k = 1, best = -1;
  for (int64_t k = 1; k <= 64 && k <= a.B; k++) {
    const int64_t waves = ((int64_t)a.C * k + sms - 1) / sms;
    const int64_t cost = waves * ((a.B + k - 1) / k + 1);
    if (best < 0 || cost < best) best = cost, best_k = k;
  }
  p->ctas_per_channel = (int)best_k;
  return true;
}

template <int S, int MT, int NWS>
static cudaError_t launch_tcl_t(const FwdArgs& a, const TclPlan& p, cudaStream_t st) {
  auto k = prnet_fwd_tcl_kernel<S, MT, NWS>;
  cudaError_t e =
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)p.ctas_per_channel, (unsigned)a.C);
  k<<<grid, 32 * (NWS + 1), p.smem_bytes, st>>>(a, p.ly, p.ctas_per_channel);
  return cudaGetLastError();
}

template <int S, int NWS>
static cudaError_t launch_tcl_m(const FwdArgs& a, const TclPlan& p, cudaStream_t st) {
  return p.mt == 1   ? launch_tcl_t<S, 1, NWS>(a, p, st)
         : p.mt == 2 ? launch_tcl_t<S, 2, NWS>(a, p, st)
                     : launch_tcl_t<S, 4, NWS>(a, p, st);
}

cudaError_t launch_tcl_kernel(const FwdArgs& a, const TclPlan& p, cudaStream_t st) {
  switch (a.S) {
    case 12: return p.nws == 8 ? launch_tcl_m<12, 8>(a, p, st) : launch_tcl_m<12, 16>(a, p, st);
    case 24: return p.nws == 8 ? launch_tcl_m<24, 8>(a, p, st) : launch_tcl_m<24, 16>(a, p, st);
    case 48: return launch_tcl_m<48, 16>(a, p, st);
    case 96: return launch_tcl_m<96, 16>(a, p, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace prnet
