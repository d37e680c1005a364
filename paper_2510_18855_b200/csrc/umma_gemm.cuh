// umma_gemm.cuh -- persistent, warp-specialised tcgen05 GEMM for sm_100a with the
// three epilogues the IcePop path needs:
//
//   EPI_STORE : C (+)= A.B^T   -> f32 / bf16 (grad_hidden K4, grad_weight K5)
//   EPI_LSE   : Z = A.B^T / T  -> per-(row, n-tile) online (max, sum-exp, sum p*z) partials
//               plus the gathered logit of the sampled token; Z never leaves TMEM (K1).
//               Replaces batched_train_logits + batched_log_softmax (policy.py:279-289,
//               350-355) and the gather lp_cur = log_probs[pos, tok] (objective.py:223).
//   EPI_DZ    : recompute Z tile, dZ = c_t * (e_{y_t} - softmax(z_t)) -> bf16 (K3),
//               objective.py:250-252.
//
// Tile: BM = 128 rows (one TMEM lane per row), BN = 256 columns, BK = 64 (one 128-byte
// swizzle atom of bf16). Roles (192 threads, 1 CTA / SM):
//   warp 0      : TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1      : TMEM allocator + MMA issuer (one elected lane), 2 TMEM accumulators
//   warps 2..5  : epilogue; thread i of warp w owns TMEM lane 32*(w%4)+i == tile row.
// The accumulator is double-buffered in TMEM (2 x 256 of the 512 columns) so the
// epilogue of tile i overlaps the MMAs of tile i+1.
#pragma once

#include "sm100.cuh"

namespace icp {

constexpr int BM = 128;
constexpr int BK = 64;
// Warp roles: 0 = TMA producer, 1 = MMA issuer (+ tile scheduler), 2.. = epilogue. K1 (EPI_LSE)
// runs two epilogue warps per TMEM lane quarter, each on half of the tile's columns: its
// softmax epilogue is exp2-throughput and latency bound, and a second warp per SM sub-partition
// roughly halves its time (it must hide behind -- or, on 512-wide tiles, partly expose -- the
// next tile's MMAs). The other epilogues use one warp per quarter.
__host__ __device__ constexpr int epi_warps(int epi) { return epi == 1 /*EPI_LSE*/ ? 8 : 4; }
__host__ __device__ constexpr int gemm_threads(int epi) { return 64 + 32 * epi_warps(epi); }
constexpr float LOG2E_F = 1.4426950408889634f;
// Stored probabilities: slabs whose maximum (log2 units) lies within +-PROBS_REF_RANGE are
// stored as 2^u (reference 0), so Q.W and Q^T.H' stay finite (|q| <= 2^60) in fp32.
constexpr float PROBS_REF_RANGE = 60.f;

// EPI_LSE_REF / EPI_DZ_REF are the KL-to-ref variants (objective.py:254-263): a second B
// operand (W_ref) shares every A (hidden) tile and accumulates into a second TMEM accumulator.
enum EpiKind { EPI_STORE = 0, EPI_LSE = 1, EPI_DZ = 2, EPI_LSE_REF = 3, EPI_DZ_REF = 4 };

__host__ __device__ constexpr bool epi_dual(int epi) { return epi == EPI_LSE_REF || epi == EPI_DZ_REF; }

struct GemmShape {
  int32_t M, N, K;
  int32_t m_tiles, n_tiles, k_blocks;
  // Scheduling items: a RUN is run_len consecutive n-tiles of one m-block (fewer at the ragged
  // end), handed to one unit as a whole, so an epilogue can carry per-row state across the run
  // (K1 merges its softmax statistics over the run and writes one partial per run instead of
  // one per tile). num_tiles counts runs (= tiles when run_len == 1).
  int32_t run_len;
  int32_t num_tiles;
  int32_t group_m;       // raster: GROUP_M m-tiles walk the n dimension together (L2 reuse)
  int32_t* tile_counter;  // dynamic schedule: zeroed before launch; nullptr = static round robin
  // static schedule with a grid barrier per wave (long-K GEMMs), or nullptr. wave_counter[0]
  // counts issued k-chunks; wave_counter[1] is the abandon flag (see chunk_wait).
  int32_t* wave_counter;
  int32_t sync_kb;        // waves: k-blocks per barrier chunk (0 = one barrier per wave)
  uint32_t wave_timeout_ns;  // a barrier wait longer than this abandons the barriers of the launch
  int32_t* diag;          // device diagnostics: diag[0] += 1 per abandoned launch (or nullptr)
  // Block sparsity (device lists, or null): the GEMM runs only k-blocks kb_map[0 .. *kb_cnt)
  // of K and m-tiles mt_map[0 .. *mt_cnt) of M; the skipped ones hold only zero rows.
  const int32_t* kb_map;
  const int32_t* kb_cnt;
  const int32_t* mt_map;
  const int32_t* mt_cnt;
  // Device-side extent (sync-free compaction): if ext_dev, the M (ext_dim = 1) or K (ext_dim = 2)
  // extent is clamp(*ext_dev - ext_base, 0, static extent), read at kernel start.
  const int32_t* ext_dev;
  int32_t ext_base;
  int32_t ext_dim;
  int32_t keep_empty;  // K extent 0: still run the tiles (the epilogue stores zeros + acc_src)
  uint32_t epi_sleep_ns;  // backoff of the epilogue warps' wait for a finished accumulator
  int32_t dz_tma_store;   // EPI_DZ: stage dZ tiles in smem and write them with TMA (else direct stores)
};

__host__ __device__ __forceinline__ int n_chunks(const GemmShape& sh) {
  return (sh.n_tiles + sh.run_len - 1) / sh.run_len;
}

// Resolve a device-side extent into the shape every role of the kernel uses.
__device__ __forceinline__ void resolve_extent(GemmShape& sh, int tile_m, int bn) {
  if (!sh.ext_dev) return;
  const int e = max(0, min(*sh.ext_dev - sh.ext_base, sh.ext_dim == 1 ? sh.M : sh.K));
  if (sh.ext_dim == 1) {
    sh.M = e;
    sh.m_tiles = (e + tile_m - 1) / tile_m;
  } else {
    sh.K = e;
    sh.k_blocks = (e + 63) / 64;
    if (sh.k_blocks == 0 && !sh.keep_empty) sh.m_tiles = 0;  // nothing to accumulate
  }
  (void)bn;
  sh.num_tiles = sh.m_tiles * n_chunks(sh);
}

// Apply the device-side block lists (block-sparse backward): fewer m-tiles / k-blocks.
__device__ __forceinline__ void resolve_sparsity(GemmShape& sh) {
  if (sh.mt_cnt) sh.m_tiles = max(0, min(*sh.mt_cnt, sh.m_tiles));
  if (sh.kb_cnt) {
    sh.k_blocks = max(0, min(*sh.kb_cnt, sh.k_blocks));
    if (sh.k_blocks == 0 && !sh.keep_empty) sh.m_tiles = 0;
  }
  sh.num_tiles = sh.m_tiles * n_chunks(sh);
}

__device__ __forceinline__ int ld_acquire_gpu(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct EpiParams {
  // EPI_STORE
  void* out;
  int64_t ldo;
  int32_t out_f32;
  int32_t accumulate;
  int32_t vec_ok;  // 16-byte aligned rows -> vector stores
  // EPI_LSE / EPI_DZ
  float scale_log2;        // log2(e) / T
  float inv_t;             // 1 / T
  const int32_t* targets;  // [M] sampled token ids
  float* part;             // EPI_LSE: [n_tiles][3][M] (max2, sum, q) in log2 units
  float* ztok;             // EPI_LSE: [M] z[y] (natural units), written by the owning tile
  const float* lse;        // EPI_DZ: [M] natural units
  const float* coeff;      // EPI_DZ: [M]
  const double* lp_cur;    // EPI_DZ / EPI_DZ_REF: [M] log p_y, or null: the sampled entry is c (1 - p_y)
                           // with 1 - p_y = -expm1(lp_cur) instead of c - c p_y (cancellation)
  float coeff_scale;       // EPI_DZ: grad_scale
  __nv_bfloat16* dz;       // EPI_DZ: [M, ldz]
  int64_t ldz;
  int32_t zero_rows_to;    // EPI_DZ: rows in [M, zero_rows_to) of the last tile are written as 0
  const int32_t* row_index;  // EPI_STORE: output row of GEMM row m is row_index[m] (scatter), or null
  // EPI_STORE fused reduce-scatter (dW over NVLink peer memory): output row m belongs to rank
  // o = m / rs_shard_rows and is stored into rs_slots[o] at slot row rs_rank * rs_shard_rows +
  // (m - o * rs_shard_rows), plus acc_src[m, :] (this rank's earlier-chunk partial) if given.
  int32_t rs_world;
  int32_t rs_rank;
  int64_t rs_shard_rows;
  float* rs_slots[8];
  const float* acc_src;
  // EPI_DZ_REF
  const float* lse_ref;    // [M] natural units
  const float* kl;         // [M] kl_t
  const float* kl_w;       // [M] w_t * gamma / T
  // EPI_STORE row-scaled mode (dH from the stored probabilities): out[m, n] = row_scale[m] * acc
  // + oh_coef[m] * W(oh_tok[m], n), W(y, n) at oh_w[y * oh_sy + n * oh_sn]
  const float* row_scale;
  const float* oh_coef;
  const int32_t* oh_tok;
  const __nv_bfloat16* oh_w;
  int64_t oh_sy, oh_sn;
  // EPI_LSE stored-probabilities mode: q[m, v] = 2^(u - R) as bf16 through the tensor map (row
  // stride = N), tile_max[m * tm_ld + 4 n_blk + c] = R of 64-column slab c (0 unless its
  // maximum leaves +-PROBS_REF_RANGE, then that maximum; log2 units)
  __nv_bfloat16* probs;
  float* tile_max;
  int32_t tm_ld;
};

// CG = 1: one CTA computes a 128 x BN tile (cta_group::1).
// CG = 2: a CTA pair computes a 256 x BN tile with cta_group::2 MMAs issued by the leader;
//         each CTA stages its own 128 rows of A and half (BN/2 rows) of B, so the B operand
//         is read from L2 once per pair instead of once per CTA.
// Epilogues that stage bf16 tiles in smem for TMA stores: K3's dZ and K1's stored probabilities.
__host__ __device__ constexpr bool epi_staging(int epi) { return epi == EPI_DZ || epi == EPI_LSE || epi == EPI_LSE_REF; }

// DUAL (the KL-to-ref variants): the vocabulary tile is BN = 128 wide and its B operand is the
// concatenation [W rows n0..n0+127 ; W_ref rows n0..n0+127], so ONE N = 256 MMA per k16 step
// writes z to accumulator columns [0, 128) and z_ref to [128, 256) -- the smem traffic per FLOP
// of a plain 256-wide tile (two N = 128 MMAs would read the A tile twice). With CTA pairs the
// leader stages the W half and the peer the W_ref half; a single CTA stages both.
template <int BN, int CG, bool DUAL = false, bool EPI_STAGING = false>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_ROWS_CTA = DUAL ? (CG == 2 ? BN : 2 * BN) : BN / CG;  // B rows this CTA stages
  static constexpr int B_BYTES = B_ROWS_CTA * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (220 * 1024 / STAGE_BYTES) < 6 ? (220 * 1024 / STAGE_BYTES) : 6;
  static constexpr int NACC = DUAL ? 2 : 1;              // accumulators per tile
  // double-buffered accumulators while they fit the 512 TMEM columns; 512-wide tiles (long-K
  // GEMMs, where one tile's MMAs take milliseconds and the epilogue microseconds) use one
  static constexpr int ACC_BUFS = 2 * BN * NACC <= 512 ? 2 : 1;
  static constexpr int TMEM_COLS = ACC_BUFS * BN * NACC;
  // MMAs per k16 step: N <= 256 per tcgen05.mma, so a 512-wide tile issues two, the second
  // reading B at +B_SUB_BYTES (its rows in each CTA's slab) into TMEM columns [256, 512)
  static constexpr int NSUB = BN > 256 ? BN / 256 : 1;
  static constexpr int N_MMA = DUAL ? 2 * BN : BN / NSUB;
  static constexpr int B_SUB_BYTES = (N_MMA / CG) * 128;  // K-major: rows x 128 B; MN-major: boxes x 8 KB
  static constexpr int TILE_M = BM * CG;
  static constexpr int RING = 4;  // tile-index ring (dynamic scheduler -> all roles of the pair)
  // TMA-store staging (32 rows x 128 B, SWIZZLE_128B per buffer): EPI_DZ 4 epilogue warps x 2
  // buffers, EPI_LSE 8 warps x 1 buffer
  static constexpr int EPI_BUF_BYTES = 32 * 128;
  static constexpr int EPI_STAGE_BYTES = EPI_STAGING ? 8 * EPI_BUF_BYTES : 0;
  // K1's half-merge exchange (one (max, sum, q) triple per TMEM lane), after the barrier block
  static constexpr int XCH_BYTES = EPI_STAGING ? BM * 3 * 4 : 0;
  static constexpr size_t SMEM = 1024 /*align slack*/ + (size_t)STAGES * STAGE_BYTES + EPI_STAGE_BYTES + 256 + XCH_BYTES;
};

// Run `run` -> its m-block, first n-tile and tile count. Raster: group_m m-blocks walk the n
// dimension together in chunks of run_len n-tiles (L2 reuse of both operands).
__device__ __forceinline__ void run_coords(const GemmShape& sh, int run, int& m_blk, int& n_first, int& count) {
  const int nc = n_chunks(sh);
  const int group = sh.group_m * nc;
  const int g = run / group;
  const int first_m = g * sh.group_m;
  const int gm = min(sh.m_tiles - first_m, sh.group_m);
  const int r = run - g * group;
  m_blk = first_m + r % gm;
  n_first = (r / gm) * sh.run_len;
  count = min(sh.run_len, sh.n_tiles - n_first);
  if (sh.mt_map) m_blk = __ldg(sh.mt_map + m_blk);
}

// ------------------------------------------------------------------ epilogues
// Output column of TMEM column tc of a tile whose n range starts at n0. With CTA pairs and a
// 512-wide tile each CTA stages a contiguous 256-row slab of B; MMA h (columns [256h, 256h+256))
// reads rows [128h, 128h+128) of both slabs, so its column j is B row (j / 128) * 256 + 128h + j % 128.
template <int BN, int CG>
__host__ __device__ constexpr int tile_col(int n0, int tc) {
  if (CG == 2 && BN > 256) {
    const int h = tc >> 8, j = tc & 255;
    return n0 + (j >> 7) * 256 + h * 128 + (j & 127);
  }
  return n0 + tc;
}

template <int BN, int CG>
__device__ __forceinline__ void epi_store(const GemmShape& sh, const EpiParams& ep, int m0, int n0,
                                          int row, uint32_t taddr) {
  const int mm = m0 + row;
  const bool row_ok = mm < sh.M;
  const int m = (row_ok && ep.row_index) ? __ldg(ep.row_index + mm) : mm;
  const float rs = (row_ok && ep.row_scale) ? __ldg(ep.row_scale + mm) : 1.f;
  const float oc = (row_ok && ep.oh_coef) ? __ldg(ep.oh_coef + mm) : 0.f;
  const __nv_bfloat16* wrow = oc != 0.f ? ep.oh_w + (int64_t)__ldg(ep.oh_tok + mm) * ep.oh_sy : nullptr;
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    float v[32];
    tmem_ld32(taddr + c * 32, v);  // warp-collective: never inside a per-thread branch
    const int col0 = tile_col<BN, CG>(n0, c * 32);
    if (!row_ok || col0 >= sh.N) continue;
    const bool full = (col0 + 32 <= sh.N) && ep.vec_ok;
    if (sh.k_blocks == 0) {  // empty K extent (keep_empty): TMEM was never written
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = 0.f;
    }
    if (ep.row_scale) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] *= rs;
      if (wrow) {
        if (ep.oh_sn == 1 && col0 + 32 <= sh.N) {  // [V,d] weight: 32 contiguous bf16 = 4 x 16 B
          const uint4* w4 = reinterpret_cast<const uint4*>(wrow + col0);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const uint4 x = __ldg(w4 + q4);
            const uint32_t* xw = reinterpret_cast<const uint32_t*>(&x);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xw[i]));
              v[8 * q4 + 2 * i] = fmaf(oc, f.x, v[8 * q4 + 2 * i]);
              v[8 * q4 + 2 * i + 1] = fmaf(oc, f.y, v[8 * q4 + 2 * i + 1]);
            }
          }
        } else {
#pragma unroll 4
          for (int j = 0; j < 32; ++j)
            if (col0 + j < sh.N) v[j] = fmaf(oc, __bfloat162float(wrow[(int64_t)(col0 + j) * ep.oh_sn]), v[j]);
        }
      }
    }
    if (ep.rs_world > 0) {
      const int64_t o = m / ep.rs_shard_rows;
      float* dst = ep.rs_slots[o] + ((int64_t)ep.rs_rank * ep.rs_shard_rows + (m - o * ep.rs_shard_rows)) * ep.ldo + col0;
      const float* src = ep.acc_src ? ep.acc_src + (int64_t)m * ep.ldo + col0 : nullptr;
      if (full) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4 x = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          if (src) {
            const float4 p = *reinterpret_cast<const float4*>(src + j);
            x.x += p.x; x.y += p.y; x.z += p.z; x.w += p.w;
          }
          *reinterpret_cast<float4*>(dst + j) = x;  // NVLink store into the owner's slot
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col0 + j < sh.N) dst[j] = src ? src[j] + v[j] : v[j];
      }
      continue;
    }
    if (ep.out_f32) {
      float* dst = reinterpret_cast<float*>(ep.out) + (int64_t)m * ep.ldo + col0;
      if (full) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          if (ep.accumulate) {
            const float4 p = *reinterpret_cast<const float4*>(dst + j);
            o.x += p.x; o.y += p.y; o.z += p.z; o.w += p.w;
          }
          *reinterpret_cast<float4*>(dst + j) = o;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col0 + j < sh.N) dst[j] = ep.accumulate ? dst[j] + v[j] : v[j];
      }
    } else {
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(ep.out) + (int64_t)m * ep.ldo + col0;
      if (full) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          uint4 o;
          o.x = pack_bf16x2(v[j], v[j + 1]);
          o.y = pack_bf16x2(v[j + 2], v[j + 3]);
          o.z = pack_bf16x2(v[j + 4], v[j + 5]);
          o.w = pack_bf16x2(v[j + 6], v[j + 7]);
          *reinterpret_cast<uint4*>(dst + j) = o;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col0 + j < sh.N) dst[j] = __float2bfloat16_rn(v[j]);
      }
    }
  }
}

// Stage one warp's 32 rows x 64 columns of packed bf16 (pk[0..31] = this lane's row) in a
// SWIZZLE_128B smem buffer and store it with one TMA bulk tensor store issued by lane 0. Two
// buffers per warp alternate; the store that last read a buffer must be done reading it.
// With NBUF = 1 the warp waits for its previous store to finish reading the buffer (the other
// warp on the sub-partition keeps it busy meanwhile).
template <int NBUF = 2>
__device__ __forceinline__ void stage_store_slab(const CUtensorMap* tmC, uint8_t* stage2, int& ebuf,
                                                 const uint32_t (&pk)[32], int col0, int row0, int lane) {
  uint8_t* buf = stage2 + (NBUF == 2 ? ebuf : 0) * (32 * 128);
  if (lane == 0) {
    if (NBUF == 2) bulk_wait_read<1>();
    else bulk_wait_read<0>();
  }
  __syncwarp();
  // row `lane` of the slab: 8 x 16-byte chunks, chunk k at position k ^ (lane & 7) (SWIZZLE_128B)
  const uint32_t rowp = smem_u32(buf) + lane * 128;
#pragma unroll
  for (int k = 0; k < 8; ++k) sts128(rowp + ((k ^ (lane & 7)) << 4), pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(tmC, smem_u32(buf), col0, row0);
    bulk_commit();
  }
  ebuf ^= 1;
}

// One 64-column slab of K1's epilogue (FULL: all 64 columns < N, else the first `valid`):
// slab maximum mx (log2 units), reference R, partial sums (s, q) against mx as two float2 lanes,
// and the packed bf16 q = 2^(u - R). EXCL (the rare slab holding some lane's sampled token, at
// column `rel`): s leaves that column out, so that K2 holds sum_{v != y} exactly and 1 - p_y is
// not formed by cancellation (K2 adds 2^(u_y - M) back for the log-sum-exp); q keeps it, and
// ey = 2^(u_y - mx) is returned (0 for lanes whose token is elsewhere) for the merges' rebasing.
template <bool FULL, bool EXCL>
__device__ __forceinline__ void lse_slab(float (&v)[64], int valid, float scale_log2, float& mx, float& ref,
                                         float2& sum2, float2& q2, uint32_t (&pk)[32], int rel, float& ey) {
  if (!FULL) {
#pragma unroll
    for (int j = 0; j < 64; ++j) v[j] = j < valid ? v[j] : -1e30f;
  }
  float t[22];
#pragma unroll
  for (int i = 0; i < 21; ++i) t[i] = fmax3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
  t[21] = v[63];
  float u[8];
#pragma unroll
  for (int i = 0; i < 7; ++i) u[i] = fmax3(t[3 * i], t[3 * i + 1], t[3 * i + 2]);
  u[7] = t[21];
  mx = fmax3(fmax3(u[0], u[1], u[2]), fmax3(u[3], u[4], u[5]), fmax3(u[6], u[7], u[7])) *
       scale_log2;  // scale > 0: max commutes with it
  // stored q = 2^(u - R): R = 0 while the slab maximum is within [-PROBS_REF_RANGE, +..] (one
  // scale per row then turns q into probabilities), else R = the slab maximum (exception)
  ref = fabsf(mx) <= PROBS_REF_RANGE ? 0.f : mx;
  const float qs = exp2f(mx - ref);
  const float2 qs2 = make_float2(qs, qs);
  const float2 sc2 = make_float2(scale_log2, scale_log2);
  const float2 nmx = make_float2(-mx, -mx);
  float2 sa = make_float2(0.f, 0.f), sb = sa, qa = sa, qb = sa;
  ey = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    // masked columns: d ~ -1e30 -> e = 0 and e * d = -0. All exponentials on the MUFU (6% busy
    // at this tile rate): moving every third pair to an FMA-pipe polynomial measured 0.2% slower
    // under the power cap, every other pair 0.3% (profiles/r02_ab_exp_mix.log)
    const float2 d = __ffma2_rn(make_float2(v[2 * j], v[2 * j + 1]), sc2, nmx);
    const float2 e = make_float2(fast_exp2(d.x), fast_exp2(d.y));
    const float2 es = EXCL ? make_float2(2 * j == rel ? 0.f : e.x, 2 * j + 1 == rel ? 0.f : e.y) : e;
    if (EXCL) ey = 2 * j == rel ? e.x : (2 * j + 1 == rel ? e.y : ey);
    if (j & 1) {
      sb = __fadd2_rn(sb, es);
      qb = __ffma2_rn(e, d, qb);
    } else {
      sa = __fadd2_rn(sa, es);
      qa = __ffma2_rn(e, d, qa);
    }
    const float2 p = __fmul2_rn(e, qs2);
    pk[j] = pack_bf16x2(p.x, p.y);
  }
  sum2 = __fadd2_rn(sa, sb);
  q2 = __fadd2_rn(qa, qb);
}

// K1 epilogue: log-sum-exp statistics of half of this tile's BN columns (`half`: TMEM columns
// [half BN/2, (half+1) BN/2)) for one row, in log2 units,
//   mx = max_j u_j,  s = sum_{j != y} 2^(u_j - mx),  q = sum_j 2^(u_j - mx) (u_j - mx),  u = z log2(e),
// so that, with S the merged s plus K2's 2^(u_y - M), lse = ln2 (M + log2 S), entropy =
// ln2 (log2 S - Q / S) and 1 - p_y = s / S without cancellation (K2); the halves' triples are
// merged per run (below). Rebasing q to a new maximum needs the FULL sum (s + 2^(u_y - mx) when
// the sampled token is in the range): the warp carries run_ey = 2^(u_y - run_m) (0 until it
// meets the token), and a partial holding the token stores its s with the sign bit set, so the
// next merge (half merge, K2) knows to add 2^(u_y - m) (u_y = ztok log2 e) before rebasing. One TMEM pass in 64-column slabs: each slab's
// (max, sum, q) is taken against the slab's own maximum and merged online. In
// stored-probabilities mode (ep.probs) the slab also emits q[m, v] = 2^(u_v - R) as bf16 (TMA
// stores, clipped to M rows / N columns) and tile_max[m, v / 64] = R, the slab's reference: 0
// while its maximum is within +-PROBS_REF_RANGE, else that maximum. The backward needs no logit
// recompute: for rows whose references are all 0 the probabilities are q 2^(-lse2), one scale
// per row. The statistics are the same bits in both modes.
// 512-wide tiles (one accumulator, SPLIT): the MMA warp may start the next tile's first-half
// MMAs once TMEM columns [0, 256) are read, so both warps of a quarter first read two slabs of
// that half each (then arrive on `half_bar`) and only then two of the second half: `half` then
// selects slabs {2 half, 2 half + 1, 4 + 2 half, 5 + 2 half}, output slabs 4 half .. 4 half + 3.
// Runs: (run_m, run_s, run_q) is this warp's running triple over the tiles of the current run
// (reset by the caller at the run's first tile). At the run's last tile the two warps of a TMEM
// lane quarter merge their triples through `xch` (the second-half warp hands its triple over
// between two named barriers) and the first-half warp writes partial part_idx = the run's
// n-chunk: one partial per row and run instead of two per tile.
template <int BN, int CG>
__device__ __forceinline__ void epi_lse(const GemmShape& sh, const EpiParams& ep, const CUtensorMap* tmC,
                                        uint8_t* stage1, int m0, int n0, int part_idx, bool last, int half, int row,
                                        int lane, int quarter, uint32_t taddr, uint32_t half_bar, float& run_m,
                                        float& run_s, float& run_q, float& run_ey, float* xch) {
  static_assert(BN == 256 || BN == 512, "64-column slabs, four or eight per tile");
  constexpr int NH = BN / 128;  // slabs per warp
  const int m = m0 + row;
  const bool row_ok = m < sh.M;
  const int y = (row_ok && ep.targets) ? __ldg(ep.targets + m) : -1;
  const int row0 = m0 + quarter * 32;
  const bool warp_rows = row0 < sh.M;  // warp-uniform
  const bool store = ep.probs != nullptr;
  float refs[NH];
  int ebuf = 0;
#pragma unroll
  for (int i = 0; i < NH; ++i) {
    const int c = NH == 4 ? (i < 2 ? 2 * half + i : 2 + 2 * half + i) : half * NH + i;  // TMEM slab
    if (NH == 4 && i == 2 && half_bar != 0u) {  // TMEM columns [0, BN/2): read by both warps
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_tmem_free(half_bar);
    }
    // (a software-pipelined variant loading slab i+1 during slab i measured no faster with two
    // warps per quarter, and its 128 live registers exceed the 168 available at 320 threads)
    float v[64];
    tmem_ld32(taddr + c * 64, *reinterpret_cast<float(*)[32]>(v));
    tmem_ld32(taddr + c * 64 + 32, *reinterpret_cast<float(*)[32]>(v + 32));
    refs[i] = 0.f;
    const int col0 = tile_col<BN, CG>(n0, c * 64);
    if (col0 < sh.N) {  // warp-uniform
      const int rel = y - col0;
      const bool y_slab = __any_sync(0xffffffffu, (unsigned)rel < 64u);  // some row's sampled token (rare)
      if (y_slab) {
        float zt = 0.f;
#pragma unroll
        for (int j = 0; j < 64; ++j) zt = (j == rel) ? v[j] : zt;
        if (row_ok && (unsigned)rel < 64u) ep.ztok[m] = zt * ep.inv_t;
      }
      float mx, ref, ey;
      float2 sum2, q2;
      uint32_t pk[32];
      // the ragged last slab (columns past N take no part) and the slab with a sampled token
      // are separate, warp-uniform paths so the common one carries no per-column predicates
      if (col0 + 64 <= sh.N) {
        if (y_slab) lse_slab<true, true>(v, 64, ep.scale_log2, mx, ref, sum2, q2, pk, rel, ey);
        else lse_slab<true, false>(v, 64, ep.scale_log2, mx, ref, sum2, q2, pk, -1, ey);
      } else {
        lse_slab<false, true>(v, sh.N - col0, ep.scale_log2, mx, ref, sum2, q2, pk, rel, ey);
      }
      if (store && warp_rows) stage_store_slab<1>(tmC, stage1, ebuf, pk, col0, row0, lane);
      const float s = sum2.x + sum2.y, q = q2.x + q2.y;
      refs[i] = ref;
      // merge the slab into the warp's running (max, sum, q, ey); q rebases with the full sums
      const float nm = fmaxf(run_m, mx);
      const float a = fast_exp2(run_m - nm), b = fast_exp2(mx - nm);
      run_q = fmaf(a, fmaf(run_m - nm, run_s + run_ey, run_q), b * fmaf(mx - nm, s + ey, q));
      run_s = fmaf(a, run_s, b * s);
      run_ey = fmaf(a, run_ey, b * ey);
      run_m = nm;
    }
    __syncwarp();  // the next slab's tcgen05.ld is warp-collective (.sync.aligned)
  }
  if (last) {  // warp-uniform: both warps of the quarter reach it on the same tile
    // the second-half warp's s carries its has-the-token flag in the sign bit (-0 for s = 0)
    float* x = xch + (quarter * 32 + lane) * 3;
    if (half == 1) {
      x[0] = run_m;
      x[1] = run_ey > 0.f ? -run_s : run_s;
      x[2] = run_q;
    }
    named_bar_sync(1 + quarter, 64);  // also orders ep.ztok[m] (either warp's store) before the read
    if (half == 0 && row_ok) {
      const float m2 = x[0], s2r = x[1], q2 = x[2];
      const float s2 = fabsf(s2r);
      const float ey2 = signbit(s2r) ? exp2f(ep.ztok[m] * LOG2E_F - m2) : 0.f;
      const float nm = fmaxf(run_m, m2);
      const float a = fast_exp2(run_m - nm), b = fast_exp2(m2 - nm);
      const float ps = fmaf(a, run_s, b * s2);
      float* p = ep.part + (int64_t)part_idx * 3 * sh.M + m;
      p[0] = nm;
      p[sh.M] = (run_ey > 0.f || ey2 > 0.f) ? -ps : ps;
      p[2 * (int64_t)sh.M] = fmaf(a, fmaf(run_m - nm, run_s + run_ey, run_q), b * fmaf(m2 - nm, s2 + ey2, q2));
    }
    named_bar_sync(1 + quarter, 64);  // the exchange slot is free for the next run
  }
  if (row_ok) {
    if (store) {
      // references in output-column order: TMEM slabs c, c+1 (c even) hold output slabs k, k+1
      float* tm = ep.tile_max + (int64_t)m * ep.tm_ld + n0 / 64;
#pragma unroll
      for (int i = 0; i < NH; i += 2) {
        const int c = NH == 4 ? (i < 2 ? 2 * half + i : 2 + 2 * half + i) : half * NH + i;
        const int k = tile_col<BN, CG>(0, c * 64) / 64;
        if (n0 / 64 + k + 2 <= ep.tm_ld) *reinterpret_cast<float2*>(tm + k) = make_float2(refs[i], refs[i + 1]);
      }
    }
  }
}

// The sampled token's dZ entry c (1 - p_y) from the forward's lp_cur (fp64 -expm1, exact however
// close p_y is to 1), or NAN when lp_cur is not given (then dz_entry forms c - c p_y).
__device__ __forceinline__ float sampled_dz(const EpiParams& ep, int m, bool live, float cf) {
  return (live && ep.lp_cur) ? (float)((double)cf * -expm1(__ldg(ep.lp_cur + m))) : __int_as_float(0x7fc00000);
}

__device__ __forceinline__ float dz_entry(float cf, float p, bool is_y, float dzy) {
  return is_y ? (dzy == dzy ? dzy : fmaf(-cf, p, cf)) : -cf * p;
}

// bf16 dZ of 32 columns (v: their logits), packed in pairs: -cf p, and for the lane whose
// sampled token sits at column `rel` of them its exact entry. Y (warp-uniform: some lane's token
// is in these columns, rare) selects the variant with the per-column compare; the common one
// has none (it measured 45% of K3's time at C1's short K, where the epilogue is exposed).
template <bool Y>
__device__ __forceinline__ void dz_pack32(const float* v, float scale_log2, float lse2, float cf, int rel,
                                          float dzy, bool live, uint32_t* pk) {
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const float p0 = fast_exp2(fmaf(v[2 * j], scale_log2, -lse2));
    const float p1 = fast_exp2(fmaf(v[2 * j + 1], scale_log2, -lse2));
    const float d0 = Y ? dz_entry(cf, p0, 2 * j == rel, dzy) : -cf * p0;
    const float d1 = Y ? dz_entry(cf, p1, 2 * j + 1 == rel, dzy) : -cf * p1;
    pk[j] = live ? pack_bf16x2(d0, d1) : 0u;
  }
}

// dZ = coeff_scale * c_t * (e_{y_t} - softmax(z_t)) for this tile -> bf16.
template <int BN>
__device__ __forceinline__ void epi_dz(const GemmShape& sh, const EpiParams& ep, int m0, int n0,
                                       int row, uint32_t taddr) {
  const int m = m0 + row;
  // rows past the (device-side) extent but inside the buffer are written as zeros, so a
  // reduction over rows (K5) never reads stale data in the last k-block
  const bool row_ok = m < sh.M || m < ep.zero_rows_to;
  const bool live = m < sh.M;
  const float lse2 = live ? __ldg(ep.lse + m) * LOG2E_F : 0.f;
  const float cf = live ? __ldg(ep.coeff + m) * ep.coeff_scale : 0.f;
  const int y = live ? __ldg(ep.targets + m) : -1;
  const float dzy = sampled_dz(ep, m, live, cf);
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    float v[32];
    tmem_ld32(taddr + c * 32, v);
    const int col0 = n0 + c * 32;
    const int rel = y - col0;
    const bool y_here = __any_sync(0xffffffffu, (unsigned)rel < 32u);  // warp-uniform, before lanes part
    if (!row_ok || col0 >= sh.N) continue;
    uint32_t pk[16];
    if (y_here) dz_pack32<true>(v, ep.scale_log2, lse2, cf, rel, dzy, live, pk);
    else dz_pack32<false>(v, ep.scale_log2, lse2, cf, rel, dzy, live, pk);
    __nv_bfloat16* dst = ep.dz + (int64_t)m * ep.ldz + col0;
    if (col0 + 32 <= sh.N && ep.vec_ok) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        reinterpret_cast<uint4*>(dst)[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&pk[j]);
        if (col0 + 2 * j < sh.N) dst[2 * j] = h.x;
        if (col0 + 2 * j + 1 < sh.N) dst[2 * j + 1] = h.y;
      }
    }
  }
}

// dZ epilogue with TMA stores: per 64-column slab the warp stages its 32 rows x 128 B
// (SWIZZLE_128B, conflict-free 16-byte smem stores) and lane 0 issues one bulk tensor store;
// two staging buffers per warp alternate. Rows past the device-side extent but inside the
// tensor map (< zero_rows_to) are stored as zeros; the tensor map clips rows >= zero_rows_to
// and columns >= V.
template <int BN>
__device__ __forceinline__ void epi_dz_tma(const GemmShape& sh, const EpiParams& ep, const CUtensorMap* tmC,
                                           uint8_t* stage2, int& ebuf, int m0, int n0, int row, int lane,
                                           int quarter, uint32_t taddr) {
  const int m = m0 + row;
  const bool live = m < sh.M;
  const float lse2 = live ? __ldg(ep.lse + m) * LOG2E_F : 0.f;
  const float cf = live ? __ldg(ep.coeff + m) * ep.coeff_scale : 0.f;
  const int y = live ? __ldg(ep.targets + m) : -1;
  const float dzy = sampled_dz(ep, m, live, cf);
  const int row0 = m0 + quarter * 32;  // first row of this warp's slab
  const bool warp_rows = row0 < ep.zero_rows_to;  // warp-uniform: any of its rows inside the map
#pragma unroll 1
  for (int c = 0; c < BN / 64; ++c) {
    float v[32], w[32];
    tmem_ld32(taddr + c * 64, v);
    tmem_ld32(taddr + c * 64 + 32, w);
    const int col0 = n0 + c * 64;
    if (!warp_rows || col0 >= sh.N) continue;  // warp-uniform
    uint32_t pk[32];
    const int rel = y - col0;
    if (__any_sync(0xffffffffu, (unsigned)rel < 32u)) dz_pack32<true>(v, ep.scale_log2, lse2, cf, rel, dzy, live, pk);
    else dz_pack32<false>(v, ep.scale_log2, lse2, cf, rel, dzy, live, pk);
    if (__any_sync(0xffffffffu, (unsigned)(rel - 32) < 32u))
      dz_pack32<true>(w, ep.scale_log2, lse2, cf, rel - 32, dzy, live, pk + 16);
    else
      dz_pack32<false>(w, ep.scale_log2, lse2, cf, rel - 32, dzy, live, pk + 16);
    stage_store_slab(tmC, stage2, ebuf, pk, col0, row0, lane);
  }
}

// One 32-column chunk of epi_lse_ref against the running maxima nm (z) and nr (z_ref): sums
// s (leaving out column ry, the lane's sampled token, when EXCL: its e is returned in ey),
// q = sum e d, x = sum e (u - ur), sr = sum 2^(ur - nr).
template <bool EXCL>
__device__ __forceinline__ void ref_chunk32(const float* vh, const float* wh, float nm, float nr, int ry, float& sm,
                                            float& q, float& x, float& sr, float& ey) {
  sm = 0.f, q = 0.f, x = 0.f, sr = 0.f, ey = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float d = vh[j] - nm;
    const float e = fast_exp2(d);
    if (EXCL) {
      sm += j == ry ? 0.f : e;
      ey = j == ry ? e : ey;
    } else {
      sm += e;
    }
    q = fmaf(e, d, q);
    x = fmaf(e, vh[j] - wh[j], x);
    sr += fast_exp2(wh[j] - nr);
  }
}

// KL-to-ref forward epilogue: as epi_lse for z (accumulator 0) plus, for z_ref (accumulator
// 1 = TMEM column + BN), the ref online (max, sum) and the cross term
// x = sum_j 2^(u_j - mx) (u_j - ur_j), u = z log2(e): after the merge,
// sum_v p_v (z_v - zr_v) = ln2 * X / S and kl = that - lse + lse_ref (objective.py:257-258).
// In stored-probabilities mode (ep.probs; gamma = 0, where the KL term is a diagnostic only, as
// in train_loop's own call, scheduler.py:530-542) it also writes q = 2^(u - R) per 64-column
// slab and the slab references R exactly as epi_lse does, so the backward is the stored mode's
// and the call executes one extra forward GEMM (z_ref) instead of a forward plus a recompute.
// As in epi_lse, s leaves the sampled token out (run_ey carries it for rebasing q) and a
// partial holding the token sets the sign bit of its s.
template <int BN>
__device__ __forceinline__ void epi_lse_ref(const GemmShape& sh, const EpiParams& ep, const CUtensorMap* tmC,
                                            uint8_t* stage2, int& ebuf, int m0, int n0, int n_blk, int row, int lane,
                                            int quarter, uint32_t taddr) {
  static_assert(BN % 64 == 0, "64-column slabs");
  const int m = m0 + row;
  const bool row_ok = m < sh.M;
  const int y = (row_ok && ep.targets) ? __ldg(ep.targets + m) : -1;
  const int row0 = m0 + quarter * 32;
  const bool warp_rows = row0 < sh.M;  // warp-uniform
  const bool store = ep.probs != nullptr;
  float run_m = -1e30f, run_s = 0.f, run_q = 0.f, run_x = 0.f, run_ey = 0.f;
  float ref_m = -1e30f, ref_s = 0.f;
  float refs[BN / 64];
#pragma unroll 1
  for (int sl = 0; sl < BN / 64; ++sl) {
    float v[64], w[64];
    tmem_ld32(taddr + sl * 64, *reinterpret_cast<float(*)[32]>(v));
    tmem_ld32(taddr + sl * 64 + 32, *reinterpret_cast<float(*)[32]>(v + 32));
    tmem_ld32(taddr + BN + sl * 64, *reinterpret_cast<float(*)[32]>(w));
    tmem_ld32(taddr + BN + sl * 64 + 32, *reinterpret_cast<float(*)[32]>(w + 32));
    refs[sl] = 0.f;
    const int col0 = n0 + sl * 64;
    if (col0 >= sh.N) continue;  // warp-uniform
    const int rel = y - col0;
    if ((unsigned)rel < 64u) {
      float zt = 0.f;
#pragma unroll
      for (int j = 0; j < 64; ++j) zt = (j == rel) ? v[j] : zt;
      if (row_ok) ep.ztok[m] = zt * ep.inv_t;
    }
    float smx = -1e30f;
#pragma unroll
    for (int j = 0; j < 64; ++j) {
      const bool ok = col0 + j < sh.N;
      v[j] = ok ? v[j] * ep.scale_log2 : -1e30f;
      w[j] = ok ? w[j] * ep.scale_log2 : -1e30f;
      smx = fmaxf(smx, v[j]);
    }
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const float* vh = v + 32 * hh;
      const float* wh = w + 32 * hh;
      float cm = -1e30f, cr = -1e30f;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        cm = fmaxf(cm, vh[j]);
        cr = fmaxf(cr, wh[j]);
      }
      const float nm = fmaxf(run_m, cm);
      const float a = fast_exp2(run_m - nm);
      run_q = a * (run_q + (run_m - nm) * (run_s + run_ey));  // rebased with the full sum
      run_s = a * run_s;
      run_ey = a * run_ey;
      run_x = a * run_x;
      const float nr = fmaxf(ref_m, cr);
      ref_s *= fast_exp2(ref_m - nr);
      const int ry = rel - 32 * hh;
      float sm, q, x, sr, eyc;
      if (__any_sync(0xffffffffu, (unsigned)ry < 32u)) ref_chunk32<true>(vh, wh, nm, nr, ry, sm, q, x, sr, eyc);
      else ref_chunk32<false>(vh, wh, nm, nr, -1, sm, q, x, sr, eyc);
      run_s += sm;
      run_ey += eyc;
      run_q += q;
      run_x += x;
      run_m = nm;
      ref_s += sr;
      ref_m = nr;
    }
    if (store) {
      // q = 2^(u - R), R = 0 while the slab maximum lies within +-PROBS_REF_RANGE (epi_lse)
      const float R = fabsf(smx) <= PROBS_REF_RANGE ? 0.f : smx;
      refs[sl] = R;
      if (warp_rows) {
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) pk[j] = pack_bf16x2(fast_exp2(v[2 * j] - R), fast_exp2(v[2 * j + 1] - R));
        stage_store_slab(tmC, stage2, ebuf, pk, col0, row0, lane);
      }
    }
  }
  if (row_ok) {
    float* p = ep.part + (int64_t)n_blk * 6 * sh.M + m;
    p[0] = run_m;
    p[sh.M] = run_ey > 0.f ? -run_s : run_s;
    p[2 * (int64_t)sh.M] = run_q;
    p[3 * (int64_t)sh.M] = ref_m;
    p[4 * (int64_t)sh.M] = ref_s;
    p[5 * (int64_t)sh.M] = run_x;
    if (store) {
      float* tm = ep.tile_max + (int64_t)m * ep.tm_ld;
#pragma unroll
      for (int sl = 0; sl < BN / 64; ++sl)
        if (n0 / 64 + sl < ep.tm_ld) tm[n0 / 64 + sl] = refs[sl];
      if (n0 + BN >= sh.N)  // the last tile zeroes the row's padding entries
        for (int k = n0 / 64 + BN / 64; k < ep.tm_ld; ++k) tm[k] = 0.f;
    }
  }
}

// KL-to-ref backward epilogue (gamma > 0), objective.py:250-263:
//   dZ = s * [ c (e_y - p) - kw * p * ((logp - logp_ref) - kl) ],  kw = w gamma / T.
template <int BN>
__device__ __forceinline__ void epi_dz_ref(const GemmShape& sh, const EpiParams& ep, int m0, int n0,
                                           int row, uint32_t taddr) {
  const int m = m0 + row;
  const bool row_ok = m < sh.M;
  const float lse2 = row_ok ? __ldg(ep.lse + m) * LOG2E_F : 0.f;
  const float lser2 = row_ok ? __ldg(ep.lse_ref + m) * LOG2E_F : 0.f;
  const float cf = row_ok ? __ldg(ep.coeff + m) * ep.coeff_scale : 0.f;
  const float kw = row_ok ? __ldg(ep.kl_w + m) * ep.coeff_scale : 0.f;
  const float kl = row_ok ? __ldg(ep.kl + m) : 0.f;
  const int y = row_ok ? __ldg(ep.targets + m) : -1;
  const float dzy = sampled_dz(ep, m, row_ok, cf);
  constexpr float LN2 = 0.69314718055994531f;
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    float v[32], w[32];
    tmem_ld32(taddr + c * 32, v);
    tmem_ld32(taddr + BN + c * 32, w);
    const int col0 = n0 + c * 32;
    if (!row_ok || col0 >= sh.N) continue;
    uint32_t pk[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float d[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float lp2 = fmaf(v[2 * j + h], ep.scale_log2, -lse2);    // log2 p
        const float lpr2 = fmaf(w[2 * j + h], ep.scale_log2, -lser2);  // log2 p_ref
        const float p = fast_exp2(lp2);
        const float diff = (lp2 - lpr2) * LN2 - kl;
        d[h] = dz_entry(cf, p, col0 + 2 * j + h == y, dzy) - kw * p * diff;
      }
      pk[j] = pack_bf16x2(d[0], d[1]);
    }
    __nv_bfloat16* dst = ep.dz + (int64_t)m * ep.ldz + col0;
    if (col0 + 32 <= sh.N && ep.vec_ok) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        reinterpret_cast<uint4*>(dst)[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const __nv_bfloat162 hh = *reinterpret_cast<const __nv_bfloat162*>(&pk[j]);
        if (col0 + 2 * j < sh.N) dst[2 * j] = hh.x;
        if (col0 + 2 * j + 1 < sh.N) dst[2 * j + 1] = hh.y;
      }
    }
  }
}

// ------------------------------------------------------------------ mainloop
template <int BN, bool A_MN, bool B_MN, int EPI, int CG>
__global__ void __launch_bounds__(gemm_threads(EPI), 1)
    umma_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmC,
                     const GemmShape sh_in, const EpiParams ep) {
  constexpr bool DUAL = epi_dual(EPI);
  constexpr bool STAGING = epi_staging(EPI);
  using Cfg = GemmCfg<BN, CG, DUAL, STAGING>;
  // K1 on 512-wide tiles: one accumulator, released to the MMA warp in two halves
  constexpr bool SPLIT = EPI == EPI_LSE && Cfg::ACC_BUFS == 1 && Cfg::NSUB == 2;
  constexpr int EW = epi_warps(EPI);
  GemmShape sh = sh_in;
  resolve_extent(sh, Cfg::TILE_M, BN);
  resolve_sparsity(sh);
  constexpr int STAGES = Cfg::STAGES;
  constexpr int B_ROWS = BN / CG;  // rows of B staged by this CTA (DUAL: BN rows of W or W_ref each)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint8_t* sEpi = smem + STAGES * Cfg::STAGE_BYTES;  // STAGING only (1024-aligned)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + Cfg::EPI_STAGE_BYTES);
  // barrier block: full[S] empty[S] tfull[2] tempty[2] rfull[RING] | tmem_holder | ring[RING]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4 + Cfg::RING);
  int32_t* ring = reinterpret_cast<int32_t*>(tmem_holder + 1);
  float* xch = reinterpret_cast<float*>(sEpi + Cfg::EPI_STAGE_BYTES + 256);  // XCH_BYTES (K1)
  const uint32_t full0 = smem_u32(bars);
  const uint32_t empty0 = smem_u32(bars + STAGES);
  const uint32_t tfull0 = smem_u32(bars + 2 * STAGES);
  const uint32_t tempty0 = smem_u32(bars + 2 * STAGES + 2);
  const uint32_t rfull0 = smem_u32(bars + 2 * STAGES + 4);
  const uint32_t thalf0 = tempty0 + 8;  // SPLIT: tempty[1] (unused with one accumulator)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  const int unit = blockIdx.x / CG;     // CTA pair (or CTA) index
  const int n_units = gridDim.x / CG;
  const bool dynamic = sh.tile_counter != nullptr;
  // Long-K GEMMs (K4, K5): static waves of n_units tiles with a grid barrier between waves, so
  // the pairs sharing A/B slices stay within a few stages of each other in k and the slices
  // are served from L2 (a dynamic claim order desynchronises k across in-flight tiles).
  const bool waves = !dynamic && sh.wave_counter != nullptr;
  const int n_waves = (sh.num_tiles + n_units - 1) / n_units;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    if (DUAL) prefetch_tmap(&tmB2);
    if (STAGING) prefetch_tmap(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      // Only the pair leader arrives (with expect_tx covering BOTH CTAs' TMA bytes); the peer's
      // loads just complete_tx on it. A per-k-block remote arrive from the peer would cost a
      // GPU-scope fence (MEMBAR.ALL.GPU) per stage and halved throughput when measured.
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tfull0 + 8 * s, 1);
      // one arrive per epilogue warp of the pair (SPLIT's thalf, s = 1, likewise)
      mbar_init(tempty0 + 8 * s, EW * CG);
    }
    for (int s = 0; s < Cfg::RING; ++s) mbar_init(rfull0 + 8 * s, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    if (CG == 2) {
      tmem_alloc_cg2(smem_u32(tmem_holder), Cfg::TMEM_COLS);
      tmem_relinquish_cg2();
    } else {
      tmem_alloc(smem_u32(tmem_holder), Cfg::TMEM_COLS);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  // Run sequence of this unit (a run is run_len tiles; run_len = 1 for every GEMM but K1).
  // Static: unit, unit + n_units, ... Dynamic: the leader's MMA thread claims runs from a
  // global counter (one run of prefetch) and publishes run j in ring slot j % RING -- locally
  // with st.shared + arrive, to the peer CTA with st.async (complete_tx on the peer's rfull
  // barrier, armed by the peer's producer). Run j+2 is published only after the MMA has waited
  // for the epilogue of the tile two accumulators back (a tile of run j-1 or earlier), so a slot
  // is never overwritten while a role of either CTA may still read it. -1 ends the sequence.
  auto ring_get = [&](int j, bool arm) -> int {
    if (!dynamic) {
      const int t = unit + j * n_units;
      return t < sh.num_tiles ? t : -1;
    }
    const int s = j & (Cfg::RING - 1);
    if (arm) mbar_arrive_expect_tx(rfull0 + 8 * s, 4);
    mbar_wait(rfull0 + 8 * s, (uint32_t)(j / Cfg::RING) & 1u);
    return *reinterpret_cast<volatile int32_t*>(ring + s);
  };

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs of a pair load their own halves)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      // Waves are split into k-chunks of `skb` k-blocks: no unit issues the loads of chunk g
      // before every unit has issued those of chunk g-1 (one monotonic counter over the whole
      // launch; skb = k_blocks is a plain barrier per wave). This keeps the tiles of a wave
      // within ~2 chunks of each other in k, so the operand slices they share stay in L2 even
      // when K is long (K5: K = tokens). The barrier is a locality hint, not a correctness
      // requirement: the grid is sized to fit an idle GPU, but a concurrent kernel (an NCCL
      // kernel on a comm stream, another stream, an MPS neighbour) can hold SMs so that some
      // units start only after others finish. A unit that waits longer than wave_timeout_ns
      // (normally ~50 us per chunk) therefore sets the abandon flag, and from then on no unit
      // of the launch waits: the GEMM completes with the same result, only without the L2
      // alignment. It never spins forever.
      const int skb = (sh.sync_kb > 0 && sh.sync_kb < sh.k_blocks) ? sh.sync_kb : max(sh.k_blocks, 1);
      const int spt = max(1, (sh.k_blocks + skb - 1) / skb);  // chunks per tile
      volatile int32_t* abandon = sh.wave_counter ? sh.wave_counter + 1 : nullptr;
      auto chunk_wait = [&](int g) {
        const int target = n_units * g;
        if (*abandon) return;
        const uint64_t t0 = globaltimer_ns();
        while (ld_acquire_gpu(sh.wave_counter) < target) {
          __nanosleep(256);
          if (*abandon) return;
          if (globaltimer_ns() - t0 > sh.wave_timeout_ns) {
            if (atomicExch(const_cast<int32_t*>(abandon), 1) == 0 && sh.diag) atomicAdd(sh.diag, 1);
            return;
          }
        }
      };
      for (int j = 0;; ++j) {
        const int tile = ring_get(j, CG == 2 && rank == 1);
        if (tile < 0) {
          if (waves && rank == 0 && n_waves > j) atomicAdd(sh.wave_counter, (n_waves - j) * spt);  // pre-pay
          break;
        }
        if (waves && rank == 0 && sh.k_blocks == 0) {  // empty K extent: one chunk without loads
          chunk_wait(j * spt);
          atomicAdd(sh.wave_counter, 1);
        }
        int m_blk, n_first, n_count;
        run_coords(sh, tile, m_blk, n_first, n_count);
        const int m0 = m_blk * Cfg::TILE_M + (int)rank * BM;
        for (int tt = 0; tt < n_count; ++tt) {
          const int n0 = (n_first + tt) * BN + (DUAL ? 0 : (int)rank * B_ROWS);
          for (int kb = 0; kb < sh.k_blocks; ++kb) {
            if (waves && rank == 0 && kb % skb == 0) chunk_wait(j * spt + kb / skb);
            const int kc = (sh.kb_map ? __ldg(sh.kb_map + kb) : kb) * BK;  // k coordinate of this block
            mbar_wait(empty0 + 8 * stage, phase ^ 1);
            const uint32_t fb_local = full0 + 8 * stage;
            const uint32_t a_dst = smem_u32(sA + stage * Cfg::A_BYTES);
            const uint32_t b_dst = smem_u32(sB + stage * Cfg::B_BYTES);
            if (CG == 1) {
              mbar_arrive_expect_tx(fb_local, Cfg::STAGE_BYTES);
              if (!A_MN) {
                tma_load_2d(a_dst, &tmA, fb_local, kc, m0);
              } else {
#pragma unroll
                for (int j2 = 0; j2 < BM / 64; ++j2) tma_load_2d(a_dst + j2 * (BK * 128), &tmA, fb_local, m0 + 64 * j2, kc);
              }
              // DUAL: the W_ref rows follow the W rows (K-major: BN rows x 128 B; MN-major: BN/64 boxes)
              constexpr uint32_t b2_off = B_MN ? (BN / 64) * (BK * 128) : BN * 128;
              if (!B_MN) {
                tma_load_2d(b_dst, &tmB, fb_local, kc, n0);
                if (DUAL) tma_load_2d(b_dst + b2_off, &tmB2, fb_local, kc, n0);
              } else {
#pragma unroll
                for (int j2 = 0; j2 < (DUAL ? BN : B_ROWS) / 64; ++j2) {
                  tma_load_2d(b_dst + j2 * (BK * 128), &tmB, fb_local, n0 + 64 * j2, kc);
                  if (DUAL) tma_load_2d(b_dst + b2_off + j2 * (BK * 128), &tmB2, fb_local, n0 + 64 * j2, kc);
                }
              }
            } else {
              const uint32_t fb = mapa_shared(fb_local, 0);  // the leader's barrier counts both halves
              if (rank == 0) mbar_arrive_expect_tx(fb_local, CG * Cfg::STAGE_BYTES);
              if (!A_MN) {
                tma_load_2d_cg2(a_dst, &tmA, fb, kc, m0);
              } else {
#pragma unroll
                for (int j2 = 0; j2 < BM / 64; ++j2) tma_load_2d_cg2(a_dst + j2 * (BK * 128), &tmA, fb, m0 + 64 * j2, kc);
              }
              // DUAL: the leader stages the tile's W rows, the peer the same rows of W_ref
              const CUtensorMap* tb = (DUAL && rank == 1) ? &tmB2 : &tmB;
              if (!B_MN) {
                tma_load_2d_cg2(b_dst, tb, fb, kc, n0);
              } else {
#pragma unroll
                for (int j2 = 0; j2 < Cfg::B_ROWS_CTA / 64; ++j2)
                  tma_load_2d_cg2(b_dst + j2 * (BK * 128), tb, fb, n0 + 64 * j2, kc);
              }
            }
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
            if (waves && rank == 0 && (kb % skb == skb - 1 || kb == sh.k_blocks - 1)) atomicAdd(sh.wave_counter, 1);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (the pair leader only) + dynamic tile scheduler
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = idesc_bf16(BM * CG, Cfg::N_MMA, A_MN, B_MN);
      auto publish = [&](int j, int tile) {
        const int s = j & (Cfg::RING - 1);
        ring[s] = tile;
        mbar_arrive(rfull0 + 8 * s);
        if (CG == 2) st_async_b32(mapa_shared(smem_u32(ring + s), 1), (uint32_t)tile, mapa_shared(rfull0 + 8 * s, 1));
      };
      auto claim = [&]() -> int { return n_units + atomicAdd(sh.tile_counter, 1); };
      // cur = tile j, nxt1 = tile j+1 (already published), claimed = next claimed index
      int cur, nxt1 = -1, claimed = sh.num_tiles;
      if (dynamic) {
        cur = unit < sh.num_tiles ? unit : -1;
        publish(0, cur);
        const int t1 = cur >= 0 ? claim() : sh.num_tiles;
        nxt1 = t1 < sh.num_tiles ? t1 : -1;
        publish(1, nxt1);
        claimed = nxt1 >= 0 ? claim() : sh.num_tiles;
      } else {
        cur = ring_get(0, false);
      }
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int j = 0; cur >= 0; ++j) {
        int m_blk_r, n_first_r, n_count;
        run_coords(sh, cur, m_blk_r, n_first_r, n_count);
        (void)m_blk_r;
        (void)n_first_r;
        int nxt2 = -1;
        for (int tt = 0; tt < n_count; ++tt) {
          // SPLIT: wait only for the epilogue to have read TMEM columns [0, BN/2) (thalf)
          mbar_wait(SPLIT ? thalf0 : tempty0 + 8 * acc, acc_phase ^ 1);
          tc_fence_after();
          if (dynamic && tt == 0) {
            // the epilogue is done with the tile two accumulators back (run j-1 or earlier), so
            // every role has read run j-2's ring slot -> slot (j+2) % RING is free
            nxt2 = (nxt1 >= 0 && claimed < sh.num_tiles) ? claimed : -1;
            publish(j + 2, nxt2);
            claimed = nxt2 >= 0 ? claim() : sh.num_tiles;
          }
          const uint32_t d_tmem = tmem_base + acc * BN * Cfg::NACC;
          // MMAs of k-block kb on smem stage st for sub-tiles [h0, h1)
          auto issue = [&](int kb, int st, int h0, int h1) {
            const uint32_t a_base = smem_u32(sA + st * Cfg::A_BYTES);
            const uint32_t b_base = smem_u32(sB + st * Cfg::B_BYTES);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t ad = A_MN ? sdesc_sw128(a_base + kk * 2048, BK * 128, 1024)
                                       : sdesc_sw128(a_base + kk * 32, 16, 1024);
              const uint64_t bd = B_MN ? sdesc_sw128(b_base + kk * 2048, BK * 128, 1024)
                                       : sdesc_sw128(b_base + kk * 32, 16, 1024);
              const uint32_t accum = (kb | kk) != 0 ? 1u : 0u;
#pragma unroll
              for (int h = 0; h < Cfg::NSUB; ++h) {
                if (h < h0 || h >= h1) continue;
                // +h * B_SUB_BYTES in the start-address field (>> 4) of the descriptor
                const uint64_t bdh = bd + (uint64_t)((h * Cfg::B_SUB_BYTES) >> 4);
                if (CG == 2) umma_bf16_cg2(d_tmem + h * Cfg::N_MMA, ad, bdh, idesc, accum);
                else umma_bf16(d_tmem + h * Cfg::N_MMA, ad, bdh, idesc, accum);
              }
            }
          };
          // SPLIT: the first-half MMAs of the first `pre` k-blocks run while the epilogue still
          // reads the previous tile's second half; their stages stay full until the second-half
          // MMAs (issued once the whole accumulator is free) have read them too.
          const int pre = SPLIT ? min(STAGES, sh.k_blocks) : 0;
          if (SPLIT) {
            int st2 = stage;
            uint32_t ph2 = phase;
            for (int kb = 0; kb < pre; ++kb) {
              mbar_wait(full0 + 8 * st2, ph2);
              tc_fence_after();
              issue(kb, st2, 0, 1);
              if (++st2 == STAGES) { st2 = 0; ph2 ^= 1; }
            }
            mbar_wait(tempty0, acc_phase ^ 1);
            tc_fence_after();
          }
          for (int kb = 0; kb < sh.k_blocks; ++kb) {
            if (kb >= pre) {
              mbar_wait(full0 + 8 * stage, phase);
              tc_fence_after();
            }
            issue(kb, stage, kb < pre ? 1 : 0, Cfg::NSUB);
            // frees the smem slot (in both CTAs) when these MMAs finish
            if (CG == 2) umma_commit_cg2(empty0 + 8 * stage, 0x3); else umma_commit(empty0 + 8 * stage);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          // accumulator ready for the epilogue warps (of both CTAs)
          if (CG == 2) umma_commit_cg2(tfull0 + 8 * acc, 0x3); else umma_commit(tfull0 + 8 * acc);
          if (++acc == Cfg::ACC_BUFS) { acc = 0; acc_phase ^= 1; }
        }
        if (dynamic) {
          cur = nxt1;
          nxt1 = nxt2;
        } else {
          cur = ring_get(j + 1, false);
        }
      }
    }
  } else {
    // ---------------- epilogue warps: this CTA's 128 rows of the pair tile (EW = 8: warps
    // 2-5 take the first half of the columns, 6-9 the second; a warp reads TMEM lanes of its
    // quarter warp % 4)
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int ehalf = EW == 8 ? (warp - 2) >> 2 : 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int ebuf = 0;  // STAGING: which of this warp's two staging buffers is next
    (void)ebuf;
    for (int j = 0;; ++j) {
      const int tile = ring_get(j, false);
      if (tile < 0) break;
      int m_blk, n_first, n_count;
      run_coords(sh, tile, m_blk, n_first, n_count);
      const int m0 = m_blk * Cfg::TILE_M + (int)rank * BM;
      float run_m = -1e30f, run_s = 0.f, run_q = 0.f, run_ey = 0.f;  // EPI_LSE: this warp's run state
      (void)run_m; (void)run_s; (void)run_q; (void)run_ey;
      for (int tt = 0; tt < n_count; ++tt) {
        const int n_blk = n_first + tt;
        mbar_wait_sleep(tfull0 + 8 * acc, acc_phase, sh.epi_sleep_ns);
        tc_fence_after();
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN * Cfg::NACC;
        if constexpr (EPI == EPI_STORE) epi_store<BN, CG>(sh, ep, m0, n_blk * BN, row, taddr);
        if constexpr (EPI == EPI_LSE)
          epi_lse<BN, CG>(sh, ep, &tmC, sEpi + (warp - 2) * Cfg::EPI_BUF_BYTES, m0, n_blk * BN,
                          n_first / sh.run_len, tt == n_count - 1, ehalf, row, lane, quarter, taddr,
                          SPLIT ? (CG == 2 ? mapa_shared(thalf0, 0) : thalf0) : 0u, run_m, run_s, run_q, run_ey, xch);
        if constexpr (EPI == EPI_DZ) {
          if (sh.dz_tma_store)
            epi_dz_tma<BN>(sh, ep, &tmC, sEpi + quarter * 2 * Cfg::EPI_BUF_BYTES, ebuf, m0, n_blk * BN, row, lane,
                           quarter, taddr);
          else
            epi_dz<BN>(sh, ep, m0, n_blk * BN, row, taddr);
        }
        if constexpr (EPI == EPI_LSE_REF)
          epi_lse_ref<BN>(sh, ep, &tmC, sEpi + quarter * 2 * Cfg::EPI_BUF_BYTES, ebuf, m0, n_blk * BN, n_blk, row, lane,
                          quarter, taddr);
        if constexpr (EPI == EPI_DZ_REF) epi_dz_ref<BN>(sh, ep, m0, n_blk * BN, row, taddr);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_tmem_free(CG == 2 ? mapa_shared(tempty0 + 8 * acc, 0) : tempty0 + 8 * acc);
        }
        if (++acc == Cfg::ACC_BUFS) { acc = 0; acc_phase ^= 1; }
      }
    }
    if (EPI == EPI_STORE && ep.rs_world > 0) __threadfence_system();  // peer stores visible system-wide
    if (STAGING && lane == 0) bulk_wait<0>();  // all staged tile stores complete
  }
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (CG == 2) tmem_dealloc_cg2(tmem_base, Cfg::TMEM_COLS);
    else tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace icp
