// aux_kernels.cu -- support kernels outside the timed forward:
//   * prnet_gather_segments_kernel: seg[b][c][n][t] = x[b][c][r + n S + t]
//     (Def 2 / reading A2) -- the bit-exact index-map check of step a1;
//   * the deterministic fp64 error reduction feeding the NCCL all-reduce of
//     MSE / MAE.
#include "prnet_internal.cuh"

namespace prnet {

__global__ void prnet_gather_segments_kernel(const float* __restrict__ x, int64_t total_series,
                                             int L, int S, int N, int r, float* __restrict__ seg) {
  const int64_t per = (int64_t)N * S;
  const int64_t n_out = total_series * per;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_out;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = k / per;
    const int64_t e = k - s * per;  // = n S + t
    seg[k] = x[s * L + r + e];
  }
}

cudaError_t launch_gather_segments(const float* x, int64_t B, int C, int L, int S, int N, int r,
                                   float* seg, cudaStream_t st) {
  const int64_t total = B * (int64_t)C;
  int64_t work = total * N * S;
  int grid = (int)((work + 255) / 256);
  if (grid > 65535 * 8) grid = 65535 * 8;
  if (grid < 1) grid = 1;
  prnet_gather_segments_kernel<<<grid, 256, 0, st>>>(x, total, L, S, N, r, seg);
  return cudaGetLastError();
}

// Stage 1: partial k reduces the contiguous chunk [k*n/P, (k+1)*n/P) in a fixed
// order (thread-strided, then a fixed shared-memory tree).  Stage 2: one block
// adds the P partials in index order.  No atomics: bitwise reproducible.
__global__ void prnet_err_partial_kernel(const float* __restrict__ y, const float* __restrict__ t,
                                         int64_t n, double* __restrict__ partials) {
  __shared__ double s_sse[256], s_sae[256];
  const int64_t P = gridDim.x;
  const int64_t lo = n * blockIdx.x / P, hi = n * (blockIdx.x + 1) / P;
  double sse = 0.0, sae = 0.0;
  for (int64_t k = lo + threadIdx.x; k < hi; k += blockDim.x) {
    const double d = (double)y[k] - (double)t[k];
    sse += d * d;
    sae += fabs(d);
  }
  s_sse[threadIdx.x] = sse;
  s_sae[threadIdx.x] = sae;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s_sse[threadIdx.x] += s_sse[threadIdx.x + o];
      s_sae[threadIdx.x] += s_sae[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = s_sse[0];
    partials[2 * blockIdx.x + 1] = s_sae[0];
  }
}

__global__ void prnet_err_final_kernel(const double* __restrict__ partials, int P, int64_t n,
                                       double* __restrict__ out3) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double sse = 0.0, sae = 0.0;
    for (int k = 0; k < P; k++) {
      sse += partials[2 * k];
      sae += partials[2 * k + 1];
    }
    out3[0] = sse;
    out3[1] = sae;
    out3[2] = (double)n;
  }
}

cudaError_t launch_error_sums(const float* y, const float* tgt, int64_t n, double* partials,
                              double* out3, cudaStream_t st) {
  prnet_err_partial_kernel<<<kErrPartials, 256, 0, st>>>(y, tgt, n, partials);
  prnet_err_final_kernel<<<1, 32, 0, st>>>(partials, kErrPartials, n, out3);
  return cudaGetLastError();
}

}  // namespace prnet
