// f64_kernels.cuh -- fp64 SIMT validation path (CUDA cores, no tensor cores).
//
// Same semantics as the bf16 tensor-core path, in the reference's precision (fp64
// everywhere) so the reference's exact-identity and finite-difference tests
// (test_objective.py) run unchanged on the GPU. Logits are materialised here: the
// validation mode trades memory for exactness and is sized for reference-scale batches.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace icp {

// C[m,n] (+)= alpha * sum_k A(m,k) B(k,n), A(m,k) = A[m*sam + k*sak], B(k,n) = B[k*sbk + n*sbn].
// 64x64 tile, 16-deep K slab, 256 threads x (4x4) outputs; each output has one owner
// and a fixed k order -> deterministic.
constexpr int F64_TM = 64, F64_TN = 64, F64_TK = 16;

__global__ void __launch_bounds__(256) k_gemm_f64(const double* __restrict__ A, int64_t sam, int64_t sak,
                                                  const double* __restrict__ B, int64_t sbk, int64_t sbn,
                                                  double* __restrict__ C, int64_t ldc, int M, int N, int K,
                                                  int accumulate) {
  __shared__ double As[F64_TK][F64_TM + 1];
  __shared__ double Bs[F64_TK][F64_TN + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * F64_TM, n0 = blockIdx.x * F64_TN;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += F64_TK) {
    for (int i = threadIdx.x; i < F64_TK * F64_TM; i += 256) {
      // consecutive threads walk the contiguous dimension of A when possible
      int kk, mm;
      if (sak == 1) { kk = i % F64_TK; mm = i / F64_TK; } else { mm = i % F64_TM; kk = i / F64_TM; }
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < K) ? A[(int64_t)m * sam + (int64_t)k * sak] : 0.0;
    }
    for (int i = threadIdx.x; i < F64_TK * F64_TN; i += 256) {
      int kk, nn;
      if (sbn == 1) { nn = i % F64_TN; kk = i / F64_TN; } else { kk = i % F64_TK; nn = i / F64_TK; }
      const int n = n0 + nn, k = k0 + kk;
      Bs[kk][nn] = (n < N && k < K) ? B[(int64_t)k * sbk + (int64_t)n * sbn] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < F64_TK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= N) continue;
      double* c = C + (int64_t)m * ldc + n;
      *c = accumulate ? *c + acc[i][j] : acc[i][j];
    }
  }
}

template <int NT>
__device__ __forceinline__ double block_sum_f64(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double r = 0.0;
  for (int w = 0; w < NT / 32; ++w) r += sh[w];
  return r;
}
template <int NT>
__device__ __forceinline__ double block_max_f64(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double r = sh[0];
  for (int w = 1; w < NT / 32; ++w) r = fmax(r, sh[w]);
  return r;
}

// Row statistics of logits (policy.py:279-289, 350-355; objective.py:223, 257-258, 274):
// z = l / T (skipped when T == 1 as the reference does), shifted = z - max z,
// lse = max + log(sum exp(shifted)), lp = shifted[y] - log s, entropy = -sum p logp,
// kl = sum p (logp - logp_ref). Z / Zref are [N, V] row-major, overwritten in place
// by z (temperature applied) so the backward can reuse them.
constexpr int F64_ROW_THREADS = 256;
__global__ void __launch_bounds__(F64_ROW_THREADS)
    k_rowstats_f64(double* __restrict__ Z, double* __restrict__ Zref, int64_t V, double temperature,
                   const int32_t* __restrict__ tokens, double* __restrict__ lse_out,
                   double* __restrict__ lp_out, double* __restrict__ ent_out,
                   double* __restrict__ kl_out, double* __restrict__ lse_ref_out,
                   unsigned* __restrict__ err_word) {
  __shared__ double sh[F64_ROW_THREADS / 32];
  const int64_t t = blockIdx.x;
  double* z = Z + t * V;
  const bool scale = temperature != 1.0;
  double mx = -INFINITY;
  bool bad = false;
  for (int64_t v = threadIdx.x; v < V; v += blockDim.x) {
    double x = z[v];
    if (scale) { x = x / temperature; z[v] = x; }
    if (!isfinite(x)) bad = true;
    mx = fmax(mx, x);
  }
  mx = block_max_f64<F64_ROW_THREADS>(mx, sh);
  double s = 0.0;
  for (int64_t v = threadIdx.x; v < V; v += blockDim.x) s += exp(z[v] - mx);
  s = block_sum_f64<F64_ROW_THREADS>(s, sh);
  const double logs = log(s);
  double ent = 0.0;
  for (int64_t v = threadIdx.x; v < V; v += blockDim.x) {
    const double sh_v = z[v] - mx;
    const double lp = sh_v - logs;
    ent += (exp(sh_v) / s) * lp;
  }
  ent = -block_sum_f64<F64_ROW_THREADS>(ent, sh);
  double kl = 0.0, lse_ref = 0.0;
  if (Zref) {
    double* zr = Zref + t * V;
    double mr = -INFINITY;
    for (int64_t v = threadIdx.x; v < V; v += blockDim.x) {
      double x = zr[v];
      if (scale) { x = x / temperature; zr[v] = x; }
      if (!isfinite(x)) bad = true;
      mr = fmax(mr, x);
    }
    mr = block_max_f64<F64_ROW_THREADS>(mr, sh);
    double sr = 0.0;
    for (int64_t v = threadIdx.x; v < V; v += blockDim.x) sr += exp(zr[v] - mr);
    sr = block_sum_f64<F64_ROW_THREADS>(sr, sh);
    const double logsr = log(sr);
    for (int64_t v = threadIdx.x; v < V; v += blockDim.x) {
      const double sh_v = z[v] - mx;
      const double diff = (sh_v - logs) - ((zr[v] - mr) - logsr);
      kl += (exp(sh_v) / s) * diff;
    }
    kl = block_sum_f64<F64_ROW_THREADS>(kl, sh);
    lse_ref = mr + logsr;
  }
  if (threadIdx.x == 0) {
    const int y = tokens[t];
    lse_out[t] = mx + logs;
    lp_out[t] = (z[y] - mx) - logs;
    ent_out[t] = ent;
    if (kl_out) kl_out[t] = kl;
    if (lse_ref_out) lse_ref_out[t] = lse_ref;
  }
  if (bad) atomicOr(err_word, 4u);  // ICEPOP_ERR_NONFINITE (integer OR: order-free)
}

// dZ in place over Z (which holds z = l/T):
//   dZ = s * [ coeff_t (e_y - p) - (w_t gamma / T) p (logp - logp_ref - kl_t) ]
// (objective.py:250-263), s = grad_scale.
__global__ void __launch_bounds__(F64_ROW_THREADS)
    k_dz_f64(double* __restrict__ Z, const double* __restrict__ Zref, int64_t V,
             const int32_t* __restrict__ tokens, const double* __restrict__ lse,
             const double* __restrict__ lse_ref, const double* __restrict__ kl,
             const double* __restrict__ coeff, const double* __restrict__ wgamma_over_t,
             double grad_scale) {
  const int64_t t = blockIdx.x;
  double* z = Z + t * V;
  const double c = coeff[t];
  const double l = lse[t];
  const int y = tokens[t];
  const double kg = (Zref && wgamma_over_t) ? wgamma_over_t[t] : 0.0;
  for (int64_t v = threadIdx.x; v < V; v += blockDim.x) {
    const double logp = z[v] - l;
    const double p = exp(logp);
    double g = -c * p;
    if (v == y) g += c;
    if (kg != 0.0) {
      const double logpr = Zref[t * V + v] - lse_ref[t];
      g -= kg * (p * ((logp - logpr) - kl[t]));
    }
    z[v] = grad_scale * g;
  }
}

// w_t * gamma / T per token (objective.py:259), computed from the batch geometry.
__global__ void k_kl_weight_f64(const int32_t* __restrict__ cu_seqlens, int32_t n_seqs,
                                const int32_t* __restrict__ group_offsets, int32_t n_groups,
                                int64_t token_offset, int64_t n_tokens, double gamma,
                                double temperature, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tokens) return;
  const int64_t tg = token_offset + t;
  int lo = 0, hi = n_seqs + 1;
  while (lo < hi) { const int mid = (lo + hi) >> 1; if ((int64_t)cu_seqlens[mid] <= tg) lo = mid + 1; else hi = mid; }
  const int seq = lo - 1;
  lo = 0; hi = n_groups + 1;
  while (lo < hi) { const int mid = (lo + hi) >> 1; if (group_offsets[mid] <= seq) lo = mid + 1; else hi = mid; }
  const int g = lo - 1;
  const int64_t n_i = (int64_t)cu_seqlens[seq + 1] - cu_seqlens[seq];
  const int64_t G = (int64_t)group_offsets[g + 1] - group_offsets[g];
  const double w = 1.0 / (double)((int64_t)n_groups * G * n_i);
  out[t] = w * gamma / temperature;
}

}  // namespace icp
