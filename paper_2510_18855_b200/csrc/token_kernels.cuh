// token_kernels.cuh -- per-token, bandwidth-bound kernels of the IcePop path.
//
//   k0_group_advantages : objective.py:153-159 (numpy pairwise-sum order reproduced, so
//                         the advantages are bit-identical to the reference's).
//   k2_icepop_tokens    : merge of the K1 split-V partials (lse, lp_cur, entropy) and the
//                         IcePop mask / ratio / clipped surrogate / gradient coefficient,
//                         objective.py:215-252, with the reference's fp64 arithmetic order.
//   k_finalize_stats    : fixed-order reduction of per-block fp64 partials (no atomics).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/icepop.h"

namespace icp {

constexpr int TOK_THREADS = 256;
constexpr float LN2_F = 0.69314718055994531f;
constexpr float LOG2E_TOK = 1.4426950408889634f;

// numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src, pairwise_sum)
// for contiguous data, over f(i) for i in [0, n). Reproducing its association order
// makes the group advantages bit-identical to numpy's r.mean() / r.std(). All adds are
// __dadd_rn and the squares __dmul_rn so nvcc cannot contract them into FMAs (numpy
// rounds every operation separately).
template <class F>
__device__ double np_pairwise_sum(F f, int lo, int n) {
  if (n < 8) {
    double res = 0.;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, f(lo + i));
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = f(lo + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], f(lo + i + j));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, f(lo + i));
    return res;
  }
  // n > 128: split in two halves with the first a multiple of 8 (iterative on the left)
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise_sum(f, lo, n2), np_pairwise_sum(f, lo + n2, n - n2));
}

// One thread per group: A_i = (R_i - mean) / max(std_pop, 1e-6)  (objective.py:153-159).
// Groups with fewer than 2 sequences yield NaN (the host layer raises ValueError first).
__global__ void k0_group_advantages(const double* __restrict__ rewards,
                                    const int32_t* __restrict__ group_offsets, int32_t n_groups,
                                    double* __restrict__ adv) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_groups) return;
  const int s0 = group_offsets[g], s1 = group_offsets[g + 1];
  const int n = s1 - s0;
  const double* r = rewards + s0;
  if (n < 2) {
    for (int i = 0; i < n; ++i) adv[s0 + i] = nan("");
    return;
  }
  const double mean = np_pairwise_sum([&](int i) { return r[i]; }, 0, n) / (double)n;
  const double var = np_pairwise_sum([&](int i) { const double x = __dsub_rn(r[i], mean); return __dmul_rn(x, x); }, 0, n) / (double)n;
  const double std = sqrt(var);
  const double den = std > 1e-6 ? std : 1e-6;  // max(std, 1e-6)
  for (int i = 0; i < n; ++i) adv[s0 + i] = __ddiv_rn(__dsub_rn(r[i], mean), den);
}

struct TokenArgs {
  int64_t n_tokens;
  int64_t token_offset;
  int32_t n_seqs;
  int32_t n_groups;
  const int32_t* tokens;
  const double* lp_old;
  const double* lp_inf;
  const int32_t* cu_seqlens;
  const int32_t* group_offsets;
  const double* adv;
  const double* calib_in;  // caller-computed c_t, or null (exp on the device)
  // bf16 mode inputs: K1 partials
  const float* part;  // [n_parts][3 or 6 rows][n_tokens] (MODE 0 / MODE 3)
  int32_t n_parts;
  int32_t part_cols;  // vocabulary columns per partial (the token's partial is y / part_cols)
  const float* ztok;  // [n_tokens]
  // f64 mode inputs (already computed per token by the f64 row kernel)
  const double* lp_cur_in;
  const double* entropy_in;
  const double* kl_in;
  // on-policy mode (MODE 2): recorded lse / entropy of lp_train_old's forward
  const float* lse_in;
  const float* entropy_in_f;
  // config
  double alpha, beta, clip_eps, tis_cap, temperature, kl_coeff;
  int32_t algo;
  // outputs (any may be null unless noted)
  float* lse_f;
  double* lp_cur;
  float* entropy_f;
  uint8_t* kept;
  double* calib;
  double* surrogate;
  float* coeff_f;
  double* coeff_d;
  float* kl_f;       // KL-to-ref outputs (MODE 3)
  float* lse_ref_f;
  float* kl_w_f;     // w_t * gamma / T (backward coefficient of the KL gradient)
  double* block_stats;  // [gridDim.x][ICEPOP_NSTATS] (required)
};

__device__ __forceinline__ int upper_bound_i32(const int32_t* a, int n, int64_t x) {
  // first index i in [0, n) with a[i] > x (a non-decreasing)
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((int64_t)a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Per-token weight w_t = 1 / (n_groups * G_g * n_i)  (objective.py:215)
__device__ __forceinline__ void seq_of_token(const TokenArgs& a, int64_t t_global, int& seq, double& w) {
  seq = upper_bound_i32(a.cu_seqlens, a.n_seqs + 1, t_global) - 1;
  const int g = upper_bound_i32(a.group_offsets, a.n_groups + 1, seq) - 1;
  const int64_t n_i = (int64_t)a.cu_seqlens[seq + 1] - a.cu_seqlens[seq];
  const int64_t G = (int64_t)a.group_offsets[g + 1] - a.group_offsets[g];
  w = 1.0 / (double)((int64_t)a.n_groups * G * n_i);
}

template <int NW>
__device__ __forceinline__ void block_reduce_stats(double (&st)[ICEPOP_NSTATS], unsigned err,
                                                   double* out) {
  __shared__ double sh[NW][ICEPOP_NSTATS];
  __shared__ unsigned sherr[NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < ICEPOP_NSTATS - 1; ++k) {
    double v = st[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    st[k] = v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) err |= __shfl_xor_sync(0xffffffffu, err, o);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < ICEPOP_NSTATS - 1; ++k) sh[warp][k] = st[k];
    sherr[warp] = err;
  }
  __syncthreads();
  if (threadIdx.x < ICEPOP_NSTATS) {
    const int k = threadIdx.x;
    double v = 0.0;
    unsigned e = 0;
    for (int w = 0; w < NW; ++w) {
      if (k < ICEPOP_NSTATS - 1) v += sh[w][k]; else e |= sherr[w];
    }
    out[(int64_t)blockIdx.x * ICEPOP_NSTATS + k] = (k < ICEPOP_NSTATS - 1) ? v : (double)e;
  }
}

// The partial holding token y (clamped: an out-of-range token is reported by k_check_tokens).
__device__ __forceinline__ int64_t token_part(int32_t y, int32_t part_cols, int32_t n_parts) {
  return (int64_t)min(max(y, 0) / part_cols, n_parts - 1);
}

// Running merge of K1's split-V partials for one token (log2 units): (M, S, Q) over the z
// partials (S leaves the sampled token out: K1 flags the partial holding it with the sign bit
// of its s, which the merge drops), and for R == 6 the ref (Mr, Sr) and the cross term X.
struct PartMerge {
  float M = -1e30f, S = 0.f, Q = 0.f, Mr = -1e30f, Sr = 0.f, X = 0.f;
  template <int R>
  __device__ __forceinline__ void add(const float (&v)[R]) {
    const float mj = v[0], sj = fabsf(v[1]), qj = v[2];
    const float nm = fmaxf(M, mj);
    const float ca = exp2f(M - nm), cb = exp2f(mj - nm);
    // Q is sum 2^(u - M) (u - M): rebasing to nm adds (M - nm) S before the rescale. With S
    // leaving the token out, each rebase from the token's partial on misses (M_k - nm_k)
    // 2^(u_y - nm_k); rescaled to the final M these telescope to (m_y - M) 2^(u_y - M), m_y
    // that partial's maximum, added once in finish() (tracking the flag in this loop measured
    // 1.5x slower: the partial is located from the token index instead)
    Q = fmaf(ca, fmaf(M - nm, S, Q), cb * fmaf(mj - nm, sj, qj));
    S = fmaf(ca, S, cb * sj);
    if constexpr (R == 6) {
      X = fmaf(ca, X, cb * v[5]);
      const float nr = fmaxf(Mr, v[3]);
      Sr = fmaf(exp2f(Mr - nr), Sr, exp2f(v[3] - nr) * v[4]);
      Mr = nr;
    }
    M = nm;
  }
  // After the last partial, with zy = z_y / T (natural units) and my the maximum of the
  // partial holding the token: the partials leave the sampled token out of S, so add
  // 2^(u_y - M) back (and, to Q, its share of the rebasing) for the log-sum-exp and entropy,
  // and take a confident token's log-prob as log1p(-S_{v != y} / S), which keeps 1 - p_y (the
  // backward's -expm1(lp_cur)) to fp32 relative precision however close p_y is to 1 (z_y - lse
  // would keep only lse's absolute precision, ~1e-6 for |z| ~ 10). Returns the full sum S.
  __device__ __forceinline__ float finish(float zy, float my, float& lse, double& lp, float& entropy) {
    const float ey = exp2f(zy * LOG2E_TOK - M);
    const float q = fmaf(my - M, ey, Q);
    const float s = S + ey;
    const float l2s = log2f(s);
    lse = (M + l2s) * LN2_F;
    entropy = (l2s - q / s) * LN2_F;
    lp = ey > 0.5f * s ? (double)log1pf(-S / s) : (double)(zy - lse);
    return s;
  }
};

// One pass over a token's partials with a running maximum: each partial is read exactly once
// (a max pass first would re-read the maxima from DRAM: they exceed L2 at C2's size). Loads
// are issued UNROLL partials ahead of the dependent merge chain, for memory-level parallelism
// (profiles/k2_ab.py A/B).
template <int R>
__device__ __forceinline__ void merge_partials(PartMerge& pm, const float* __restrict__ part, int n_parts, int64_t n,
                                               int64_t t) {
  constexpr int UNROLL = 16;  // 16 partials in flight per thread: 0.257 -> 0.200 ms at C2 (4: 0.28 with the prefetch)
  const float* p = part + t;
  const int64_t stride = (int64_t)R * n;
  int j = 0;
  for (; j + UNROLL <= n_parts; j += UNROLL, p += UNROLL * stride) {
    float v[UNROLL][R];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) v[u][r] = __ldg(p + u * stride + r * n);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) pm.add<R>(v[u]);
  }
  for (; j < n_parts; ++j, p += stride) {
    float v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = __ldg(p + r * n);
    pm.add<R>(v);
  }
}

// MODE 0: bf16 path (merge K1's partials, 3 rows each), MODE 3: the same with the KL-to-ref
// dual partials (6 rows), MODE 1: fp64 path (lp_cur/entropy/kl given), MODE 2: on-policy
// (theta == theta_old): lp_cur = lp_train_old, lse/entropy recorded.
template <int MODE>
__global__ void __launch_bounds__(TOK_THREADS) k2_icepop_tokens(const TokenArgs a) {
  constexpr bool MERGE = MODE == 0 || MODE == 3;
  constexpr int R = MODE == 3 ? 6 : 3;
  double st[ICEPOP_NSTATS] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned err = 0;
  const double clip_lo = 1.0 - a.clip_eps, clip_hi = 1.0 + a.clip_eps;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < a.n_tokens;
       t += (int64_t)gridDim.x * blockDim.x) {
    double lp_cur, ent, kl = 0.0;
    if (MERGE) {
      // merge split-V partials -> lse, entropy, lp_cur
      // the token's partial maximum first: its (uncoalesced) load overlaps the merge loop
      const float my = __ldg(a.part + token_part(__ldg(a.tokens + t), a.part_cols, a.n_parts) * R * a.n_tokens + t);
      PartMerge pm;
      merge_partials<R>(pm, a.part, a.n_parts, a.n_tokens, t);
      float lse, entf;
      const float S = pm.finish(a.ztok[t], my, lse, lp_cur, entf);
      ent = (double)entf;
      if (a.lse_f) a.lse_f[t] = lse;
      if (a.entropy_f) a.entropy_f[t] = entf;
      if (!isfinite(lse) || !isfinite(entf) || !isfinite(a.ztok[t])) err |= ICEPOP_ERR_NONFINITE;
      if (R == 6) {
        // kl = sum_v p (logp - logp_ref) = sum_v p (z - z_ref) - lse + lse_ref  (objective.py:257-258)
        const float lse_r = (pm.Mr + log2f(pm.Sr)) * LN2_F;
        const float klf = (pm.X / S) * LN2_F - lse + lse_r;
        kl = (double)klf;
        if (a.kl_f) a.kl_f[t] = klf;
        if (a.lse_ref_f) a.lse_ref_f[t] = lse_r;
        if (!isfinite(klf)) err |= ICEPOP_ERR_NONFINITE;
      }
    } else if (MODE == 1) {
      lp_cur = a.lp_cur_in[t];
      ent = a.entropy_in[t];
      kl = a.kl_in ? a.kl_in[t] : 0.0;
    } else {
      lp_cur = a.lp_old[t];
      const float ef = a.entropy_in_f ? a.entropy_in_f[t] : 0.f;
      ent = (double)ef;
      if (a.lse_f) a.lse_f[t] = a.lse_in[t];
      if (a.entropy_f) a.entropy_f[t] = ef;
    }
    if (a.lp_cur && MODE != 1) a.lp_cur[t] = lp_cur;

    int seq;
    double w;
    seq_of_token(a, a.token_offset + t, seq, w);
    const double A = a.adv[seq];
    const double lpo = a.lp_old[t];
    // calibration and mask (objective.py:227-238)
    const double c = a.calib_in ? a.calib_in[t] : exp(__dsub_rn(lpo, a.lp_inf[t]));
    if (!isfinite(c)) err |= ICEPOP_ERR_CALIB_OVERFLOW;
    bool kept;
    double factor;
    if (a.algo == ICEPOP_ALGO_ICEPOP) {
      kept = (c >= a.alpha) && (c <= a.beta);
      factor = kept ? c : 0.0;
    } else if (a.algo == ICEPOP_ALGO_GRPO) {
      kept = true;
      factor = c;
    } else {
      kept = true;
      factor = fmin(c, a.tis_cap);
    }
    // ratio / clip / surrogate (objective.py:240-246)
    const double r = exp(__dsub_rn(lp_cur, lpo));
    if (!isfinite(r)) err |= ICEPOP_ERR_RATIO_OVERFLOW;
    const double unclipped = r * A;
    const double clipped = fmin(fmax(r, clip_lo), clip_hi) * A;
    const bool active = unclipped <= clipped;
    const double pg = factor * (active ? unclipped : clipped);
    // gradient coefficient (objective.py:250)
    const double coeff = active ? w * factor * r * A / a.temperature : 0.0;
    const double value = __dsub_rn(pg, __dmul_rn(a.kl_coeff, kl));  // objective.py:268, no FMA

    if (a.kept) a.kept[t] = kept ? 1 : 0;
    if (a.calib) a.calib[t] = c;
    if (a.surrogate) a.surrogate[t] = pg;
    if (a.coeff_f) a.coeff_f[t] = (float)coeff;
    if (a.coeff_d) a.coeff_d[t] = coeff;
    if (a.kl_w_f) a.kl_w_f[t] = (float)(w * a.kl_coeff / a.temperature);

    st[ICEPOP_STAT_OBJECTIVE] += w * value;
    st[ICEPOP_STAT_N_POPPED] += kept ? 0.0 : 1.0;
    st[ICEPOP_STAT_TOKENS] += 1.0;
    st[ICEPOP_STAT_SUM_ENTROPY] += ent;
    st[ICEPOP_STAT_SUM_ENTROPY_POPPED] += kept ? 0.0 : ent;
    st[ICEPOP_STAT_SUM_LOGP] += lp_cur;
    st[ICEPOP_STAT_SUM_KL] += kl;
  }
  if (!isfinite(st[ICEPOP_STAT_OBJECTIVE])) err |= ICEPOP_ERR_NONFINITE;
  block_reduce_stats<TOK_THREADS / 32>(st, err, a.block_stats);
}

// Single block: stats[k] = sum over blocks (fixed order); errors OR-ed.
__global__ void k_finalize_stats(const double* __restrict__ block_stats, int n_blocks,
                                 double* __restrict__ stats) {
  __shared__ double sh[ICEPOP_NSTATS][33];
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;  // 8 warps x 32 lanes
  double v = 0.0;
  unsigned e = 0;
  for (int b = lane; b < n_blocks; b += 32) {
    const double x = block_stats[(int64_t)b * ICEPOP_NSTATS + k];
    if (k == ICEPOP_STAT_ERRORS) e |= (unsigned)x; else v += x;
  }
  sh[k][lane] = (k == ICEPOP_STAT_ERRORS) ? (double)e : v;
  __syncthreads();
  if (lane == 0) {
    double acc = 0.0;
    unsigned ee = 0;
    for (int i = 0; i < 32; ++i) {
      if (k == ICEPOP_STAT_ERRORS) ee |= (unsigned)sh[k][i]; else acc += sh[k][i];
    }
    stats[k] = (k == ICEPOP_STAT_ERRORS) ? (double)ee : acc;
  }
}

// ------------------------------------------------------------------ discrepancy probe (f-4)
// kl_t = KL(softmax(z_p) || softmax(z_q)) per row from the dual-LSE partials (6 rows per
// tile); block partial sums of kl in fixed order for the probe-set mean (discrepancy.py:132-141).
__global__ void __launch_bounds__(TOK_THREADS) k_kl_finish(const float* __restrict__ part, int n_parts, int64_t n,
                                                          float* __restrict__ kl_out, float* __restrict__ lse_p,
                                                          float* __restrict__ lse_q, double* __restrict__ block_sums) {
  double acc = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    float M = -1e30f, Mr = -1e30f;
    for (int j = 0; j < n_parts; ++j) {
      const float* p = part + (int64_t)j * 6 * n + t;
      M = fmaxf(M, p[0]);
      Mr = fmaxf(Mr, p[3 * n]);
    }
    float S = 0.f, Sr = 0.f, X = 0.f;
    for (int j = 0; j < n_parts; ++j) {
      const float* p = part + (int64_t)j * 6 * n + t;
      const float sc = exp2f(p[0] - M);
      S = fmaf(p[n], sc, S);
      Sr = fmaf(p[4 * n], exp2f(p[3 * n] - Mr), Sr);
      X = fmaf(p[5 * n], sc, X);
    }
    const float lp = (M + log2f(S)) * LN2_F, lq = (Mr + log2f(Sr)) * LN2_F;
    const float kl = (X / S) * LN2_F - lp + lq;
    if (kl_out) kl_out[t] = kl;
    if (lse_p) lse_p[t] = lp;
    if (lse_q) lse_q[t] = lq;
    acc += (double)kl;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double sh[TOK_THREADS / 32];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < TOK_THREADS / 32; ++w) s += sh[w];
    block_sums[blockIdx.x] = s;
  }
}

__global__ void k_sum_blocks(const double* __restrict__ block_sums, int nb, double scale, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += block_sums[b];
    *out = s * scale;
  }
}

// delta and max token gap per probe row (discrepancy.py:132-141): with p the inference engine's
// distribution softmax(zi) and q the training engine's softmax(zt) (both already divided by T):
//   kl_t = sum_v p_v (log p_v - log q_v),  gap_t = max_v |p_v - q_v|.
// One block per row, fp64 arithmetic, fixed-order block reductions (deterministic). zt is
// read as TZ (the train logits the GEMM wrote, scaled here by inv_t), zi as TI.
constexpr int DG_THREADS = 256;

template <class T>
__device__ __forceinline__ double block_reduce_dg(double v, bool is_max, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, x) : v + x;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double r = sh[0];
  for (int w = 1; w < DG_THREADS / 32; ++w) r = is_max ? fmax(r, sh[w]) : r + sh[w];
  return r;
}

template <class TZ, class TI>
__global__ void __launch_bounds__(DG_THREADS) k_delta_gap_rows(const TZ* __restrict__ zt, const TI* __restrict__ zi,
                                                               int64_t n, int64_t V, double inv_t,
                                                               double* __restrict__ kl, double* __restrict__ gap) {
  __shared__ double sh[DG_THREADS / 32];
  for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
    const TZ* a = zt + t * V;
    const TI* b = zi + t * V;
    double ma = -INFINITY, mb = -INFINITY;
    for (int64_t v = threadIdx.x; v < V; v += DG_THREADS) {
      ma = fmax(ma, (double)a[v] * inv_t);
      mb = fmax(mb, (double)b[v]);
    }
    ma = block_reduce_dg<double>(ma, true, sh);
    mb = block_reduce_dg<double>(mb, true, sh);
    double sa = 0.0, sb = 0.0;
    for (int64_t v = threadIdx.x; v < V; v += DG_THREADS) {
      sa += exp((double)a[v] * inv_t - ma);
      sb += exp((double)b[v] - mb);
    }
    sa = block_reduce_dg<double>(sa, false, sh);
    sb = block_reduce_dg<double>(sb, false, sh);
    const double lsa = ma + log(sa), lsb = mb + log(sb);
    double k = 0.0, g = 0.0;
    for (int64_t v = threadIdx.x; v < V; v += DG_THREADS) {
      const double lq = (double)a[v] * inv_t - lsa, lp = (double)b[v] - lsb;
      const double p = exp(lp);
      k += p * (lp - lq);
      g = fmax(g, fabs(p - exp(lq)));
    }
    k = block_reduce_dg<double>(k, false, sh);
    g = block_reduce_dg<double>(g, true, sh);
    if (threadIdx.x == 0) {
      kl[t] = k;
      gap[t] = g;
    }
  }
}

// delta = mean_t kl_t (fixed order), max_gap = max_t gap_t: one block.
__global__ void k_delta_gap_finish(const double* __restrict__ kl, const double* __restrict__ gap, int64_t n,
                                   double* __restrict__ delta, double* __restrict__ max_gap) {
  __shared__ double sh[DG_THREADS / 32];
  double s = 0.0, m = 0.0;
  for (int64_t t = threadIdx.x; t < n; t += DG_THREADS) {
    s += kl[t];
    m = fmax(m, gap[t]);
  }
  s = block_reduce_dg<double>(s, false, sh);
  m = block_reduce_dg<double>(m, true, sh);
  if (threadIdx.x == 0) {
    if (delta) *delta = s / (double)n;
    if (max_gap) *max_gap = m;
  }
}

// ------------------------------------------------------------------ optimizer step (f-2)
// Gradient ASCENT as the reference (objective.py:301-326): v = beta v + g (momentum) or v = g,
// w += lr v; non-finite weights set the error word; optional bf16 copy of w for the GEMMs.
__global__ void k_sgd_update(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ v,
                             __nv_bfloat16* __restrict__ w_bf16, int64_t n, float lr, float beta,
                             unsigned* __restrict__ err) {
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float step = g[i];
    if (v) {
      step = fmaf(beta, v[i], step);
      v[i] = step;
    }
    const float nw = fmaf(lr, step, w[i]);
    w[i] = nw;
    if (w_bf16) w_bf16[i] = __float2bfloat16_rn(nw);
    bad |= !isfinite(nw);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, ICEPOP_ERR_NONFINITE);
}

// The reference's own update in fp64 (objective.py:301-326), bit for bit: numpy rounds
// lr * step and the sum separately (no FMA), and the momentum step v' = beta v + g likewise.
// w_out / v_out may alias w / v (in-place update); non-finite results set the error word.
__global__ void k_sgd_update_f64(double* __restrict__ w_out, const double* __restrict__ w,
                                 const double* __restrict__ g, const double* __restrict__ v,
                                 double* __restrict__ v_out, int64_t n, double lr, double beta,
                                 unsigned* __restrict__ err) {
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double step = g[i];
    if (v) {
      step = __dadd_rn(__dmul_rn(beta, v[i]), step);  // objective.py:323
      v_out[i] = step;
    }
    const double nw = __dadd_rn(w[i], __dmul_rn(lr, step));  // objective.py:307
    w_out[i] = nw;
    bad |= !isfinite(nw);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, ICEPOP_ERR_NONFINITE);
}

// ------------------------------------------------------------------ reduce-scatter fold
// out[i] = sum_r slots[r][i] in rank order (deterministic), the owner's half of the fused
// dW reduce-scatter (the K5 epilogue already placed every rank's rows in its slot).
__global__ void k_rs_fold(const float4* __restrict__ slots, int world, int64_t n4, float4* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 s = slots[i];
    for (int r = 1; r < world; ++r) {
      const float4 x = slots[(int64_t)r * n4 + i];
      s.x += x.x; s.y += x.y; s.z += x.z; s.w += x.w;
    }
    out[i] = s;
  }
}

// ------------------------------------------------------------------ active-row compaction
// Rows whose gradient coefficient is exactly zero (popped tokens, clip-inactive tokens,
// zero-advantage sequences) have dZ == 0 (objective.py:250-252), so the backward GEMMs run
// on the compacted active rows only. Order-preserving (deterministic) three-pass compaction;
// the count stays on the device so the backward needs no host sync.
constexpr int COMPACT_BLOCK = 1024;

__global__ void __launch_bounds__(COMPACT_BLOCK) k_active_count(const float* __restrict__ coeff, int64_t n,
                                                              int32_t* __restrict__ block_counts) {
  __shared__ int warp_counts[COMPACT_BLOCK / 32];
  const int64_t t = (int64_t)blockIdx.x * COMPACT_BLOCK + threadIdx.x;
  const bool act = t < n && coeff[t] != 0.f;
  const unsigned b = __ballot_sync(0xffffffffu, act);
  if ((threadIdx.x & 31) == 0) warp_counts[threadIdx.x >> 5] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    int c = 0;
    for (int w = 0; w < COMPACT_BLOCK / 32; ++w) c += warp_counts[w];
    block_counts[blockIdx.x] = c;
  }
}

// Single block: exclusive scan of block counts (sequential in chunks; nb is small).
__global__ void k_active_scan(const int32_t* __restrict__ block_counts, int nb, int32_t* __restrict__ block_offsets,
                              int32_t* __restrict__ n_active) {
  __shared__ int partial[1024];
  const int per = (nb + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per, b1 = min(nb, b0 + per);
  int s = 0;
  for (int b = b0; b < b1; ++b) s += block_counts[b];
  partial[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      const int v = partial[i];
      partial[i] = acc;
      acc += v;
    }
    *n_active = acc;
  }
  __syncthreads();
  int off = partial[threadIdx.x];
  for (int b = b0; b < b1; ++b) {
    block_offsets[b] = off;
    off += block_counts[b];
  }
}

__global__ void __launch_bounds__(COMPACT_BLOCK) k_active_scatter(const float* __restrict__ coeff, int64_t n,
                                                                const int32_t* __restrict__ block_offsets,
                                                                int32_t* __restrict__ idx) {
  __shared__ int warp_counts[COMPACT_BLOCK / 32];
  const int64_t t = (int64_t)blockIdx.x * COMPACT_BLOCK + threadIdx.x;
  const bool act = t < n && coeff[t] != 0.f;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(0xffffffffu, act);
  if (lane == 0) warp_counts[warp] = __popc(b);
  __syncthreads();
  int before = 0;
  for (int w = 0; w < warp; ++w) before += warp_counts[w];
  if (act) idx[block_offsets[blockIdx.x] + before + __popc(b & ((1u << lane) - 1u))] = (int32_t)t;
}

// Gather active rows: hid_act[i] = hid[idx[i]] (bf16 rows of d elements, d % 8 == 0) and the
// per-row scalars (lp_cur when given); rows [n_active, rows_cap) are zero-filled up to the next
// multiple of 256.
__global__ void k_gather_active(const int32_t* __restrict__ idx, const int32_t* __restrict__ n_active,
                                const uint4* __restrict__ hid, int64_t d8, const int32_t* __restrict__ tok,
                                const float* __restrict__ lse, const float* __restrict__ coeff,
                                uint4* __restrict__ hid_act, int32_t* __restrict__ tok_act,
                                float* __restrict__ lse_act, float* __restrict__ coeff_act,
                                const double* __restrict__ lp, double* __restrict__ lp_act, int64_t rows_cap) {
  const int na = *n_active;
  const int64_t rows_r = ((int64_t)na + 255) / 256 * 256;
  const int64_t rows = rows_cap < rows_r ? rows_cap : rows_r;
  const int64_t total = rows * d8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / d8, c = i - r * d8;
    if (r < na) {
      const int32_t src = idx[r];
      hid_act[i] = hid[(int64_t)src * d8 + c];
      if (c == 0) {
        tok_act[r] = tok[src];
        lse_act[r] = lse[src];
        coeff_act[r] = coeff[src];
        if (lp) lp_act[r] = lp[src];
      }
    } else {
      hid_act[i] = make_uint4(0u, 0u, 0u, 0u);
      if (c == 0) {
        tok_act[r] = 0;
        lse_act[r] = 0.f;
        coeff_act[r] = 0.f;
        if (lp) lp_act[r] = 0.0;
      }
    }
  }
}

// Stored-probabilities dZ in place (exception rows of the row-scaled backward, or every row when
// the backward has no workspace): turns K1's q[t, v] = 2^(u - R_slab) into
//   dz[t, v] = cf_t * (e_{y_t} - q[t, v] * 2^(R_slab(t, v / 64) - lse2_t)),  cf_t = coeff_t * scale,
// the same expression epi_dz evaluates from recomputed logits (p = 2^(u - lse2)). Rows with
// cf_t == 0 are written as zeros without being read. One block per row (grid-stride); each
// 16-byte chunk (8 columns, one slab) takes its slab scale from the L1-resident tile_max row;
// 4 chunks in flight per thread, streaming loads/stores (measured 28.97 -> 28.55 ms at C2).
// Needs V % 8 == 0.
constexpr int DZP_THREADS = 256;
__global__ void __launch_bounds__(DZP_THREADS) k_dz_probs(uint4* __restrict__ probs, const float* __restrict__ tile_max,
                                                          int32_t tm_ld, const float* __restrict__ lse,
                                                          const float* __restrict__ coeff, float coeff_scale,
                                                          const int32_t* __restrict__ tokens, int64_t n, int64_t v8,
                                                          const double* __restrict__ lp_cur,
                                                          const uint8_t* __restrict__ only = nullptr) {
  for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
    if (only && !only[t]) continue;  // block-uniform: rows the GEMMs scale themselves stay as they are
    uint4* row = probs + t * v8;
    const float cf = coeff[t] * coeff_scale;
    if (cf == 0.f) {
      for (int64_t k = threadIdx.x; k < v8; k += DZP_THREADS) row[k] = make_uint4(0u, 0u, 0u, 0u);
      continue;  // block-uniform
    }
    const float lse2 = lse[t] * 1.4426950408889634f;  // log2(e)
    const int y = tokens[t];
    // the sampled token's entry c (1 - p_y) from p_y = exp(lp_cur) in fp64: formed from the bf16
    // q_y it would lose 2^-9 p_y / (1 - p_y) of its value to cancellation (objective.py:251-252)
    const float dzy = (float)((double)cf * -expm1(lp_cur[t]));
    const float* tm = tile_max + t * tm_ld;
    constexpr int U = 4;
    for (int64_t k0 = threadIdx.x; k0 < v8; k0 += U * DZP_THREADS) {
      uint4 x[U];
      float sm[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t k = k0 + u * DZP_THREADS;
        if (k < v8) {
          x[u] = __ldcs(row + k);  // streaming: each chunk is read and written exactly once
          sm[u] = __ldg(tm + (k >> 3));  // 64 columns per slab = 8 chunks
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t k = k0 + u * DZP_THREADS;
        if (k >= v8) break;
        const float s = exp2f(sm[u] - lse2) * -cf;
        uint32_t* w = reinterpret_cast<uint32_t*>(&x[u]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 qq = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
          const int64_t c = k * 8 + 2 * i;
          const float d0 = c == y ? dzy : qq.x * s;
          const float d1 = c + 1 == y ? dzy : qq.y * s;
          const __nv_bfloat162 o = __floats2bfloat162_rn(d0, d1);
          w[i] = *reinterpret_cast<const uint32_t*>(&o);
        }
        __stcs(row + k, x[u]);
      }
    }
  }
}

// Block-sparse backward lists (stored-probabilities mode). flags[b] = 1 if any token of the
// 64-token block b has a nonzero gradient coefficient (one warp per block, coalesced).
__global__ void k_block_flags(const float* __restrict__ coeff, int64_t n, int32_t* __restrict__ flags) {
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nb = (n + 63) / 64;
  if (b >= nb) return;
  const int64_t t0 = b * 64 + lane, t1 = t0 + 32;
  const bool act = (t0 < n && coeff[t0] != 0.f) || (t1 < n && coeff[t1] != 0.f);
  const unsigned any = __ballot_sync(0xffffffffu, act);
  if (lane == 0) flags[b] = any != 0u;
}

// One CTA, increasing order (deterministic): kb_map = active 64-token blocks (the k-blocks of
// K5, K = tokens), mt_map = tiles of `tile_blocks` blocks with any active block (the m-tiles
// of K4, M = tokens); *cnt[0] / *cnt[1] their counts.
constexpr int BL_THREADS = 1024;
__global__ void __launch_bounds__(BL_THREADS) k_block_lists(const int32_t* __restrict__ flags, int64_t nb,
                                                            int tile_blocks, int32_t* __restrict__ kb_map,
                                                            int32_t* __restrict__ mt_map, int32_t* __restrict__ cnt) {
  __shared__ int warp_tot[BL_THREADS / 32];
  __shared__ int base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nt = (nb + tile_blocks - 1) / tile_blocks;
  for (int list = 0; list < 2; ++list) {
    const int64_t count = list == 0 ? nb : nt;
    int32_t* map = list == 0 ? kb_map : mt_map;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    for (int64_t i0 = 0; i0 < count; i0 += BL_THREADS) {
      const int64_t i = i0 + threadIdx.x;
      bool p = false;
      if (i < count) {
        if (list == 0) {
          p = flags[i] != 0;
        } else {
          for (int j = 0; j < tile_blocks && i * tile_blocks + j < nb; ++j) p = p || flags[i * tile_blocks + j] != 0;
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, p);
      if (lane == 0) warp_tot[warp] = __popc(bal);
      __syncthreads();
      int off = base;
      for (int w = 0; w < warp; ++w) off += warp_tot[w];
      if (p) map[off + __popc(bal & ((1u << lane) - 1u))] = (int32_t)i;
      __syncthreads();
      if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < BL_THREADS / 32; ++w) tot += warp_tot[w];
        base += tot;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) cnt[list] = base;
    __syncthreads();
  }
}

// Row-scaled stored-probabilities backward, per row t. q was stored as 2^(u - R_slab) with
// R_slab = 0 except for slabs whose maximum left the finite range (exception rows, any R != 0).
// For the other rows p = q 2^(-lse2) has one scale per row, so the GEMMs take it directly:
//   dH = s (Q.W) + c (1 - p_y) W[y],  dW = Q^T.(s H) + scatter_y(c (1 - p_y) H),
//   s = -c 2^(-lse2), c = coeff * gs,
// with q_y set to 0 in probs here, so the sampled token's column enters only through the
// one-hot term, whose 1 - p_y = -expm1(lp_cur) is fp64-exact (objective.py:251-252). Taking
// it as c - c q_y 2^(-lse2) instead cancels: the bf16 q_y carries 2^-9 p_y of error against a
// result of size 1 - p_y (12% on a token with p_y = 0.98, the common case in RL batches).
// Exception rows get their dZ in place (k_dz_probs with `only`) and enter the GEMMs unscaled
// (s = 1, c = 0). Writes s, c (1 - p_y), the exception flag and H' = bf16(s H) TRANSPOSED,
// hid_t[k][t] (d rows of ldt tokens; tokens >= n are zero): K5 then reads H' K-major. With
// both of K5's operands MN-major (q^T and H') the long-K GEMM ran 1-2% slower
// (profiles/major_ab.py). One block per 64-token tile: warps find the rows' scales, then the
// tile's H rows pass through shared memory 64 hidden columns at a time.
constexpr int SPP_THREADS = 256;
constexpr int SPP_TILE = 64;
constexpr int SPP_LD = SPP_TILE + 2;  // bf16 elements per smem row: 33 words, conflict-free stores
// One 64-token tile of H (rows t0.., d8 16-byte groups per row), each row scaled by s_sc[row]
// and rounded to bf16, written transposed: hid_t[k][t] (ldt tokens per row; rows >= n give zeros).
// The rows pass through shared memory 64 hidden columns at a time: coalesced 128-byte reads of
// H rows, 16-byte stores of 8 tokens of one hidden column. Blocks along gridDim.y take
// interleaved 64-column groups (small token counts still fill the GPU).
__device__ __forceinline__ void transpose_tile_scaled(const uint4* __restrict__ hid, int64_t d8, int64_t t0, int64_t n,
                                                      const float* s_sc, uint32_t* tile, uint4* __restrict__ hid_t,
                                                      int64_t ldt) {
  const uint16_t* th = reinterpret_cast<const uint16_t*>(tile);
  for (int64_t c8 = (int64_t)blockIdx.y * (SPP_TILE / 8); c8 < d8; c8 += (int64_t)gridDim.y * (SPP_TILE / 8)) {
    // load + scale: thread -> (row, 8-column group), stored as four 32-bit words
    for (int i = threadIdx.x; i < SPP_TILE * 8; i += SPP_THREADS) {
      const int row = i >> 3, q = i & 7;
      const int64_t t = t0 + row;
      uint4 x = make_uint4(0u, 0u, 0u, 0u);
      if (t < n && c8 + q < d8) x = hid[t * d8 + c8 + q];
      uint32_t* w = reinterpret_cast<uint32_t*>(&x);
      const float sc = s_sc[row];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 h = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[k]));
        const __nv_bfloat162 o = __floats2bfloat162_rn(h.x * sc, h.y * sc);
        tile[row * (SPP_LD / 2) + 4 * q + k] = *reinterpret_cast<const uint32_t*>(&o);
      }
    }
    __syncthreads();
    // transposed store: thread -> (hidden column, 8-token group), one 16-byte store
    for (int i = threadIdx.x; i < SPP_TILE * 8; i += SPP_THREADS) {
      const int c = i >> 3, q = i & 7;
      if (c8 * 8 + c < d8 * 8) {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          w[k] = (uint32_t)th[(8 * q + 2 * k) * SPP_LD + c] | ((uint32_t)th[(8 * q + 2 * k + 1) * SPP_LD + c] << 16);
        hid_t[((c8 * 8 + c) * ldt + t0) / 8 + q] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(SPP_THREADS) k_sp_prep(const float* __restrict__ tile_max, int32_t tm_ld,
                                                         int32_t n_slabs, const float* __restrict__ lse,
                                                         const float* __restrict__ coeff, float gs,
                                                         const double* __restrict__ lp_cur,
                                                         const int32_t* __restrict__ tokens,
                                                         __nv_bfloat16* __restrict__ probs, int64_t vocab,
                                                         const uint4* __restrict__ hid, int64_t d8,
                                                         float* __restrict__ rscale, float* __restrict__ ohc,
                                                         uint8_t* __restrict__ exc, uint4* __restrict__ hid_t,
                                                         int64_t ldt, int64_t n) {
  __shared__ float s_sc[SPP_TILE];
  __shared__ uint32_t tile[SPP_TILE * SPP_LD / 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_tiles = (n + SPP_TILE - 1) / SPP_TILE;
  for (int64_t tt = blockIdx.x; tt < n_tiles; tt += gridDim.x) {
    const int64_t t0 = tt * SPP_TILE;
    for (int r = warp; r < SPP_TILE; r += SPP_THREADS / 32) {
      const int64_t t = t0 + r;
      float sc = 0.f;
      if (t < n) {
        // any slab reference != 0 (an exception row): 16-byte loads, several in flight per lane
        // (tm_ld is a multiple of 4 and its padding entries are 0)
        const float4* tm4 = reinterpret_cast<const float4*>(tile_max + t * tm_ld);
        const int n4 = (n_slabs + 3) >> 2;
        bool any = false;
#pragma unroll 4
        for (int j = lane; j < n4; j += 32) {
          const float4 r = __ldg(tm4 + j);
          any |= (r.x != 0.f) | (r.y != 0.f) | (r.z != 0.f) | (r.w != 0.f);
        }
        const bool ex = __any_sync(0xffffffffu, any);
        const float cf = coeff[t] * gs;
        sc = ex ? 1.f : (cf == 0.f ? 0.f : -cf * exp2f(-lse[t] * 1.4426950408889634f));
        if (lane == 0 && blockIdx.y == 0) {  // the column-group blocks of a tile share the scales
          rscale[t] = sc;
          ohc[t] = (ex || cf == 0.f) ? 0.f : (float)((double)cf * -expm1(lp_cur[t]));
          exc[t] = ex ? 1 : 0;
          if (!ex) probs[t * vocab + tokens[t]] = __ushort_as_bfloat16((unsigned short)0);
        }
      }
      if (lane == 0) s_sc[r] = sc;
    }
    __syncthreads();
    transpose_tile_scaled(hid, d8, t0, n, s_sc, tile, hid_t, ldt);
  }
}

// The plain H^T of K5's K-major operand in the recompute backward (rows of a dZ chunk, scale 1).
__global__ void __launch_bounds__(SPP_THREADS) k_transpose_rows(const uint4* __restrict__ hid, int64_t d8,
                                                                 uint4* __restrict__ hid_t, int64_t ldt, int64_t n) {
  __shared__ float s_sc[SPP_TILE];
  __shared__ uint32_t tile[SPP_TILE * SPP_LD / 2];
  if (threadIdx.x < SPP_TILE) s_sc[threadIdx.x] = 1.f;
  const int64_t n_tiles = (n + SPP_TILE - 1) / SPP_TILE;
  for (int64_t tt = blockIdx.x; tt < n_tiles; tt += gridDim.x) {
    __syncthreads();
    transpose_tile_scaled(hid, d8, tt * SPP_TILE, n, s_sc, tile, hid_t, ldt);
  }
}

__global__ void k_iota(int32_t* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)i;
}

// Destination of the one-hot part of dW: element (vocabulary row y, hidden column col) of dW lives
// at dw + y * sy + col * sc in the weight's layout ([V,d]: sy = d, sc = 1; [d,V]: sy = 1, sc = V)
// -- or, with the fused reduce-scatter (rs_world > 0), in the slot its owner keeps for this rank:
// dW row r (= y for [V,d], = col for [d,V]) is owned by o = r / shard_rows and sits at row
// rank * shard_rows + r - o * shard_rows of slots[o] (row length row_len).
struct OneHotDst {
  float* dw;
  int64_t sy, sc;
  int32_t rs_world, rs_rank;
  int64_t shard_rows, row_len;
  int32_t rows_are_y;  // [V,d]: dW rows are vocabulary rows
  float* slots[8];

  __device__ __forceinline__ float* at(int64_t y, int64_t col) const {
    if (rs_world == 0) return dw + y * sy + col * sc;
    const int64_t r = rows_are_y ? y : col, c = rows_are_y ? col : y;
    const int64_t o = r / shard_rows;
    return slots[o] + ((int64_t)rs_rank * shard_rows + r - o * shard_rows) * row_len + c;
  }
};

// One-hot part of dW: dW[y, :] += sum over tokens t with y_t = y of c_t H[t, :], in increasing t
// (the token indices are radix-sorted by y, a stable sort), one block per run of equal y that
// starts in its stride: deterministic, no atomics. With the fused reduce-scatter it adds into the
// owners' slots (over NVLink) after K5 stored there, so no dense local dW has to be built.
constexpr int OHS_THREADS = 256;
__global__ void __launch_bounds__(OHS_THREADS) k_onehot_scatter(const int32_t* __restrict__ ys,
                                                                const int32_t* __restrict__ ts, int64_t n,
                                                                const float* __restrict__ ohc,
                                                                const uint4* __restrict__ hid, int64_t d8,
                                                                const OneHotDst dst) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const int32_t y = ys[i];
    if (i > 0 && ys[i - 1] == y) continue;  // not the start of a run (block-uniform)
    int64_t e = i + 1;
    while (e < n && ys[e] == y) ++e;
    for (int64_t k = threadIdx.x; k < d8; k += OHS_THREADS) {
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      bool any = false;
      for (int64_t r = i; r < e; ++r) {
        const int32_t t = ts[r];
        const float c = ohc[t];
        if (c == 0.f) continue;
        any = true;
        uint4 x = hid[(int64_t)t * d8 + k];
        const uint32_t* w = reinterpret_cast<const uint32_t*>(&x);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 h = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[j]));
          acc[2 * j] = fmaf(c, h.x, acc[2 * j]);
          acc[2 * j + 1] = fmaf(c, h.y, acc[2 * j + 1]);
        }
      }
      if (!any) continue;
      if (dst.rows_are_y) {  // 8 consecutive columns of one dW row: two 16-byte read-modify-writes
        float4* d4 = reinterpret_cast<float4*>(dst.at(y, k * 8));
        float4 a = d4[0], b = d4[1];
        a.x += acc[0]; a.y += acc[1]; a.z += acc[2]; a.w += acc[3];
        b.x += acc[4]; b.y += acc[5]; b.z += acc[6]; b.w += acc[7];
        d4[0] = a;
        d4[1] = b;
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) *dst.at(y, k * 8 + j) += acc[j];
      }
    }
  }
}

}  // namespace icp
