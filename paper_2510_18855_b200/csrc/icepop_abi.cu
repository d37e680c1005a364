// icepop_abi.cu -- extern "C" entry points of libicepop_b200.so (include/icepop.h).
//
// Host-side orchestration only: argument validation with the reference's error
// semantics, workspace carving, TMA descriptor encoding and kernel launches. All
// arithmetic runs in the kernels of umma_gemm.cuh / token_kernels.cuh / f64_kernels.cuh.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdarg>
#include <map>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include <cub/cub.cuh>

#include "../../include/icepop.h"
#include "f64_kernels.cuh"
#include "token_kernels.cuh"
#include "umma_gemm.cuh"

using namespace icp;

namespace {

constexpr uint32_t ERR_BAD_TOKEN = 8u;

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define ICP_CUDA(expr)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(ICEPOP_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),  \
                  __FILE__, __LINE__);                                                    \
  } while (0)

#define ICP_TRY(expr)            \
  do {                           \
    int _r = (expr);             \
    if (_r != ICEPOP_OK) return _r; \
  } while (0)

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Carver {
  uint8_t* base;
  size_t off = 0;
  explicit Carver(void* b) : base(static_cast<uint8_t*>(b)) {}
  template <class T>
  T* take(size_t count) {
    off = align_up(off, 256);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// ------------------------------------------------------------------ TMA descriptors
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

int encode_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
              uint32_t box_inner, uint32_t box_outer) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(ICEPOP_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(ptr) & 15u) != 0)
    return fail(ICEPOP_EINVAL, "TMA operand base must be 16-byte aligned");
  if ((ld_elems * 2) % 16 != 0)
    return fail(ICEPOP_EINVAL, "TMA operand row stride must be a multiple of 8 bf16 elements");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ICEPOP_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return ICEPOP_OK;
}

// Operand X of C = X_A . X_B^T viewed as [mn, k]:
//   K-major : stored [mn rows, k cols] with row stride ld   -> box {64, tile_mn}
//   MN-major: stored [k rows, mn cols] with row stride ld   -> box {64, 64}
int operand_map(CUtensorMap* map, const void* ptr, int64_t mn, int64_t k, int64_t ld, bool mn_major,
                int tile_mn) {
  if (!mn_major) return encode_2d(map, ptr, (uint64_t)k, (uint64_t)mn, (uint64_t)ld, 64, tile_mn);
  return encode_2d(map, ptr, (uint64_t)mn, (uint64_t)k, (uint64_t)ld, 64, 64);
}

constexpr int BN_ = 256;
constexpr int BN_WIDE = 512;

int g_cta_group = 0;  // 0 = not yet read from ICEPOP_CTA_GROUP (default 2)

// Scheduler counters (the dynamic schedule's tile counter, or the long-K waves' chunk counter
// and abandon flag): one pair per launch, zeroed stream-ordered right before it, from a ring of
// N_COUNTERS pairs per stream. Launches on one stream run in order, so a pair is reused only
// after the launch that last used it has finished; streams get their own rings (N_RINGS per
// device, assigned in order of first use and reused modulo N_RINGS beyond that). Replays of one
// captured CUDA graph on two streams at once would share pairs: replay a graph on one stream at
// a time. The pool is allocated once per device (icepop_device_check, or the first launch), so
// no allocation happens inside a stream capture.
constexpr int N_COUNTERS = 256;
constexpr int N_RINGS = 64;
struct DevicePool {
  int32_t* counters = nullptr;  // [N_RINGS][N_COUNTERS][2]
  int32_t* diag = nullptr;      // [4]: [0] launches whose wave barriers were abandoned
  unsigned next[N_RINGS] = {0};
  int n_streams = 0;
  std::map<cudaStream_t, int> ring_of;
};
DevicePool g_pool[16];
std::mutex g_counter_mutex;

int ensure_pool(int dev) {
  if (dev < 0 || dev >= 16) return fail(ICEPOP_EINVAL, "device index %d out of range", dev);
  std::lock_guard<std::mutex> lock(g_counter_mutex);
  DevicePool& p = g_pool[dev];
  if (!p.counters) {
    int32_t* buf = nullptr;
    ICP_CUDA(cudaMalloc(&buf, (2 * N_RINGS * N_COUNTERS + 4) * sizeof(int32_t)));
    ICP_CUDA(cudaMemset(buf, 0, (2 * N_RINGS * N_COUNTERS + 4) * sizeof(int32_t)));
    p.counters = buf;
    p.diag = buf + 2 * N_RINGS * N_COUNTERS;
  }
  return ICEPOP_OK;
}

int diag_ptr(int dev, int32_t** out) {
  ICP_TRY(ensure_pool(dev));
  *out = g_pool[dev].diag;
  return ICEPOP_OK;
}

// Longest a unit of a long-K GEMM waits at a wave barrier before abandoning the barriers of
// its launch (ICEPOP_WAVE_TIMEOUT_US, default 10 ms; a barrier chunk takes ~50 us at C2).
uint32_t wave_timeout_ns() {
  static uint32_t v = 0;
  if (v == 0) {
    const char* e = getenv("ICEPOP_WAVE_TIMEOUT_US");
    const long us = e ? std::max(1L, atol(e)) : 10000L;
    v = (uint32_t)std::min<long>(us * 1000L, 4000000000L);
  }
  return v;
}

int dynamic_sched() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ICEPOP_SCHED");
    v = (e && strcmp(e, "static") == 0) ? 0 : 1;
  }
  return v;
}

int long_k_blocks() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ICEPOP_LONG_K_BLOCKS");
    v = e ? std::max(1, atoi(e)) : 256;
  }
  return v;
}

int tile_counter(cudaStream_t st, int32_t** out) {
  *out = nullptr;
  if (!dynamic_sched()) return ICEPOP_OK;
  int dev = 0;
  ICP_CUDA(cudaGetDevice(&dev));
  ICP_TRY(ensure_pool(dev));
  int32_t* c = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_counter_mutex);
    DevicePool& p = g_pool[dev];
    auto it = p.ring_of.find(st);
    int ring;
    if (it == p.ring_of.end()) {
      ring = p.n_streams++ % N_RINGS;
      p.ring_of.emplace(st, ring);
    } else {
      ring = it->second;
    }
    c = p.counters + 2 * (ring * N_COUNTERS + (int)(p.next[ring]++ % N_COUNTERS));
  }
  ICP_CUDA(cudaMemsetAsync(c, 0, 2 * sizeof(int32_t), st));
  *out = c;
  return ICEPOP_OK;
}

int cta_group() {
  if (g_cta_group == 0) {
    const char* e = getenv("ICEPOP_CTA_GROUP");
    g_cta_group = (e && atoi(e) == 1) ? 1 : 2;
  }
  return g_cta_group;
}

template <int BN, bool A_MN, bool B_MN, int EPI, int CG>
int launch_umma_cg(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tb2, const CUtensorMap& tc,
                   const GemmShape& sh, const EpiParams& ep, cudaStream_t st) {
  auto kern = umma_gemm_kernel<BN, A_MN, B_MN, EPI, CG>;
  constexpr size_t smem = GemmCfg<BN, CG, epi_dual(EPI), epi_staging(EPI)>::SMEM;
  // the smem attribute is per device: one bit per device index that has it set
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  ICP_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_done.load(std::memory_order_acquire) & bit)) {
    ICP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_done.fetch_or(bit, std::memory_order_acq_rel);
  }
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.blockDim = dim3(gemm_threads(EPI));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // Persistent grid: one unit (CTA pair) per pair of SMs, capped by the clusters an idle device
  // holds at once (fewer under MPS or green contexts), so that no wave barrier waits for a
  // unit that cannot be resident.
  static std::atomic<int> max_units[16];
  int cap = num_sms() / CG;
  if (dev >= 0 && dev < 16) {
    int mu = max_units[dev].load(std::memory_order_relaxed);
    if (mu == 0) {
      cfg.gridDim = dim3((unsigned)(cap * CG));
      int n = 0;
      mu = (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n > 0) ? n : cap;
      (void)cudaGetLastError();
      max_units[dev].store(mu, std::memory_order_relaxed);
    }
    cap = std::min(cap, mu);
  }
  const int units = std::max(1, std::min(sh.num_tiles, cap));
  cfg.gridDim = dim3((unsigned)(units * CG));
  ICP_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, tb2, tc, sh, ep));
  return ICEPOP_OK;
}

template <bool A_MN, bool B_MN, int EPI>
int launch_umma(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tb2, const CUtensorMap& tc,
                const GemmShape& sh, const EpiParams& ep, cudaStream_t st, int cg, bool wide = false) {
  constexpr int BN = epi_dual(EPI) ? 128 : BN_;
  if constexpr (EPI == EPI_STORE || EPI == EPI_LSE) {
    if (wide && cg == 2) return launch_umma_cg<BN_WIDE, A_MN, B_MN, EPI, 2>(ta, tb, tb2, tc, sh, ep, st);
  }
  if (cg == 2) return launch_umma_cg<BN, A_MN, B_MN, EPI, 2>(ta, tb, tb2, tc, sh, ep, st);
  return launch_umma_cg<BN, A_MN, B_MN, EPI, 1>(ta, tb, tb2, tc, sh, ep, st);
}

// Tile raster: `group_m` m-tiles sweep the n dimension together. ICEPOP_GROUP_M overrides
// (tuning experiments); otherwise 16 tile rows (sustained-power sweep on B200: 16 beat
// 4, 8 and 32 for every GEMM of the path, see profiles/README.md).
int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? std::max(0, atoi(e)) : dflt;
}

int group_m_for(int epi, int m_tiles, int n_tiles, int cg, bool long_k, int64_t K, int units) {
  // Short K (dynamic claim order): the group's A rows stay resident in L2 while B streams, so
  // size the group for a ~32 MB A-set (measured: 16 pair-rows at K = 4096, 8 at K = 8192).
  // Long K (waves): 8 pair-rows balances A and B re-reads (measured). When a wave spans whole
  // tile rows anyway (n_tiles <= units / 2, e.g. K4/K5 with d = 4096 on 512-wide tiles), the
  // group only orders tiles inside the wave: 2 measured best (K4 1,540 -> 1,567 TFLOP/s).
  static const int g_short = env_int("ICEPOP_GROUP_M", 0);
  static const int g_long = env_int("ICEPOP_GROUP_M_LONG", 0);
  (void)epi;
  int g;
  if (long_k) {
    g = g_long > 0 ? g_long : (2 * n_tiles <= units ? 2 : 8);
  } else if (g_short > 0) {
    g = g_short;
  } else {
    const int64_t a_rows_bytes = (int64_t)BM * cg * std::max<int64_t>(K, 1) * 2;
    g = (int)std::max<int64_t>(4, std::min<int64_t>(32, (32ll << 20) / a_rows_bytes));
  }
  return std::max(1, std::min(g, m_tiles));
}

// C[M,N] = A . B^T with the given operand majors; epilogue `epi`.
struct Extent {
  const int32_t* dev = nullptr;  // device-side extent (compacted row count), or null
  int32_t base = 0;
  int32_t dim = 0;  // 1: M, 2: K
};

// BN of a GEMM with epilogue `epi` (the dual-accumulator KL variants use 128-column tiles).
inline int bn_of(int epi) { return epi_dual(epi) ? 128 : BN_; }

// Long-K plain GEMMs (K4, K5) on CTA pairs use 256 x 512 tiles (two N = 256 MMAs per k step,
// one TMEM accumulator): a third fewer operand bytes per FLOP from L2 into smem than 256 x 256
// (K1/K3 keep 256 x 256: their heavy epilogues need the double-buffered accumulator).
// ICEPOP_WIDE_TILES=0 / icepop_set_wide_tiles(0) select 256 x 256.
int g_wide_tiles = -1;

bool wide_tiles() {
  if (g_wide_tiles < 0) g_wide_tiles = std::min(env_int("ICEPOP_WIDE_TILES", 1), 2);
  return g_wide_tiles >= 1;
}

// K1 (EPI_LSE) on 256 x 512 tiles: one TMEM accumulator released to the MMA warp in halves
// (umma_gemm.cuh SPLIT). ICEPOP_K1_WIDE=1 / icepop_set_k1_wide(1) select it (CTA pairs only).
int g_k1_wide = -1;

bool k1_wide() {
  if (g_k1_wide < 0) g_k1_wide = env_int("ICEPOP_K1_WIDE", 0) ? 1 : 0;
  return g_k1_wide == 1 && cta_group() == 2;
}

// Column tile of K1.
int k1_bn() { return k1_wide() ? BN_WIDE : BN_; }

// K1's run length: the n-tiles a unit processes back to back for one m-block, merging the
// softmax statistics in registers (and the two column halves through shared memory) and writing
// one partial per row and run (umma_gemm.cuh epi_lse). Runs of 2 cut the partials K1 writes and
// K2 reads from 2 * ceil(V/256) * 12 bytes per token (3.9 GB at C2) to ceil(V/512) * 12 (0.97
// GB). Longer runs cost K1 time at C2 (measured, profiles/r02_k1_run_ab.log: 1, 2 -> 250.6,
// 251.0 ms; 4 -> 252.4; 8 -> 257.1; 16 -> 272.5 ms, one box): a pair that stays on one m-block
// for many tiles loosens the raster's sharing of each weight tile. Small problems take runs of
// 1 when fewer than 16 runs per unit would remain. ICEPOP_K1_RUN / icepop_set_k1_run override.
int g_k1_run = -1;  // 0 = automatic; ICEPOP_K1_RUN / icepop_set_k1_run

int k1_run_len(int64_t n_tokens, int64_t V, int64_t d) {
  if ((d + BK - 1) / BK >= long_k_blocks()) return 1;  // a long-K K1 runs static waves, tile by tile
  if (g_k1_run < 0) g_k1_run = env_int("ICEPOP_K1_RUN", 0);
  if (g_k1_run > 0) return std::min(g_k1_run, 64);
  const int cg = cta_group();
  const int64_t m_t = (std::max<int64_t>(n_tokens, 1) + BM * cg - 1) / (BM * cg);
  const int64_t n_t = (V + k1_bn() - 1) / k1_bn();
  const int64_t units = std::max(1, num_sms() / cg);
  int r = 2;
  while (r > 1 && m_t * ((n_t + r - 1) / r) < 16 * units) r /= 2;
  return r;
}

// Partial (max, sum, q) triples per token that K1 writes: one per run.
int64_t k1_parts(int64_t n_tokens, int64_t V, int64_t d) {
  const int64_t n_t = (V + k1_bn() - 1) / k1_bn();
  const int r = k1_run_len(n_tokens, V, d);
  return (n_t + r - 1) / r;
}

// Grid of the transposing kernels (k_sp_prep, k_transpose_rows): 64-token tiles along x and,
// when the tiles alone would not give each SM two blocks (C1: 64 tiles), 64-column groups of
// the hidden dimension along y.
dim3 spp_grid(int64_t n, int64_t d) {
  const int64_t tiles = std::max<int64_t>((n + SPP_TILE - 1) / SPP_TILE, 1);
  const int64_t groups = std::max<int64_t>((d + SPP_TILE - 1) / SPP_TILE, 1);
  const int64_t want = (2 * (int64_t)num_sms() + tiles - 1) / tiles;
  return dim3((unsigned)std::min<int64_t>(tiles, (int64_t)num_sms() * 8), (unsigned)std::max<int64_t>(1, std::min(groups, want)));
}

// Vocabulary columns per K1 partial: the sampled token y's statistics are in partial y / this.
int32_t k1_part_cols(int64_t n_tokens, int64_t V, int64_t d) { return k1_bn() * k1_run_len(n_tokens, V, d); }

// A 512-wide tile does the work of two 256-wide ones ~5% cheaper (fewer operand bytes per
// FLOP) but halves the tile count. On a small output (C1's dH: 32 wide tiles for 74 CTA
// pairs) that leaves pairs idle, so the long-K GEMMs take wide tiles only when their wave
// count costs no more than the narrow tiles' (weighted by that 5%).
bool wide_pays(int64_t M, int64_t N, int64_t units) {
  const int64_t m_t = (M + 2 * BM - 1) / (2 * BM);
  const int64_t waves_w = (m_t * ((N + BN_WIDE - 1) / BN_WIDE) + units - 1) / units;
  const int64_t waves_n = (m_t * ((N + BN_ - 1) / BN_) + units - 1) / units;
  return 2 * waves_w * 95 <= waves_n * 100;
}

// Device-side block lists of a block-sparse GEMM (GemmShape::kb_map ...), or none.
struct Sparse {
  const int32_t* kb_map = nullptr;
  const int32_t* kb_cnt = nullptr;
  const int32_t* mt_map = nullptr;
  const int32_t* mt_cnt = nullptr;
};

int run_umma(int epi, const void* A, int64_t lda, bool a_mn, const void* B, int64_t ldb, bool b_mn,
             int64_t M, int64_t N, int64_t K, EpiParams ep, cudaStream_t st, Extent ext = Extent(),
             const void* B2 = nullptr, bool keep_empty = false, Sparse sparse = Sparse()) {
  if (M <= 0 || N <= 0 || K <= 0) return ICEPOP_OK;
  if (M > INT32_MAX / 2 || N > INT32_MAX / 2 || K > INT32_MAX / 2)
    return fail(ICEPOP_EINVAL, "GEMM extent too large");
  const int cg = cta_group();
  const bool long_k = (K + BK - 1) / BK >= long_k_blocks();
  bool wide = (epi == EPI_STORE && cg == 2 && long_k && wide_tiles()) || (epi == EPI_LSE && k1_wide());
  if (wide && epi == EPI_STORE && g_wide_tiles != 2) wide = wide_pays(M, N, num_sms() / cg);
  const int bn = wide ? BN_WIDE : bn_of(epi);
  if (epi_dual(epi) && !B2) return fail(ICEPOP_EINVAL, "dual-accumulator GEMM needs a second B operand");
  CUtensorMap ta, tb, tb2;
  ICP_TRY(operand_map(&ta, A, M, K, lda, a_mn, BM));
  // B box rows: a CTA stages bn / cg rows of B; the dual-accumulator tiles stage bn rows of W
  // and of W_ref (the leader / the peer, or one CTA both: umma_gemm.cuh GemmCfg)
  const int b_box = epi_dual(epi) ? bn : bn / cg;
  ICP_TRY(operand_map(&tb, B, N, K, ldb, b_mn, b_box));
  if (B2) ICP_TRY(operand_map(&tb2, B2, N, K, ldb, b_mn, b_box));
  else tb2 = tb;
  // bf16 store map of the staging epilogues (32 rows x 64 cols boxes, SW128): EPI_DZ's dZ
  // [zero_rows_to, N] and EPI_LSE's stored probabilities [M, N]
  CUtensorMap tc = tb;
  if (epi == EPI_DZ) ICP_TRY(encode_2d(&tc, ep.dz, (uint64_t)N, (uint64_t)ep.zero_rows_to, (uint64_t)ep.ldz, 64, 32));
  if ((epi == EPI_LSE || epi == EPI_LSE_REF) && ep.probs)
    ICP_TRY(encode_2d(&tc, ep.probs, (uint64_t)N, (uint64_t)M, (uint64_t)N, 64, 32));
  GemmShape sh;
  sh.M = (int)M;
  sh.N = (int)N;
  sh.K = (int)K;
  sh.m_tiles = (int)((M + BM * cg - 1) / (BM * cg));
  sh.n_tiles = (int)((N + bn - 1) / bn);
  sh.k_blocks = (int)((K + BK - 1) / BK);
  if ((int64_t)sh.m_tiles * sh.n_tiles > INT32_MAX) return fail(ICEPOP_EINVAL, "too many tiles");
  // runs of n-tiles: K1 only (its epilogue merges statistics across a run); never with waves
  sh.run_len = (epi == EPI_LSE && !long_k) ? k1_run_len(M, N, K) : 1;
  sh.num_tiles = sh.m_tiles * n_chunks(sh);
  // static waves (with their k-chunk barrier) only when the tiles take more than one wave: a
  // single wave (C1's dH: 64 tiles for 74 pairs) ran 0.26 ms that way and 0.18 ms with the
  // dynamic schedule (the lockstep only makes every pair wait for the slowest one's loads)
  const bool waves = long_k && (int64_t)sh.m_tiles * sh.n_tiles > num_sms() / cg;
  sh.group_m = group_m_for(epi, sh.m_tiles, sh.n_tiles, cg, waves, K, num_sms() / cg);
  sh.ext_dev = ext.dim ? ext.dev : nullptr;
  sh.ext_base = ext.base;
  sh.ext_dim = ext.dim;
  sh.keep_empty = keep_empty ? 1 : 0;
  sh.kb_map = sparse.kb_map;
  sh.kb_cnt = sparse.kb_cnt;
  sh.mt_map = sparse.mt_map;
  sh.mt_cnt = sparse.mt_cnt;
  static const int sleep_ns = env_int("ICEPOP_EPI_SLEEP_NS", 0);
  sh.epi_sleep_ns = (uint32_t)sleep_ns;
  static const int dz_tma = env_int("ICEPOP_DZ_TMA_STORE", 1);
  sh.dz_tma_store = dz_tma;
  // short K: dynamic claim order keeps in-flight tiles contiguous (L2 reuse across tiles);
  // long K: static waves with a grid barrier keep in-flight tiles aligned in k.
  sh.wave_counter = nullptr;
  static const int sync_kb = env_int("ICEPOP_SYNC_KB", 64);  // K5 at C2: 1,495 -> 1,529 TFLOP/s (64 ~ 256 > 16)
  sh.sync_kb = sync_kb;
  sh.wave_timeout_ns = wave_timeout_ns();
  sh.diag = nullptr;
  if (waves) {
    ICP_TRY(tile_counter(st, &sh.wave_counter));
    sh.tile_counter = nullptr;
    int dev = 0;
    ICP_CUDA(cudaGetDevice(&dev));
    ICP_TRY(diag_ptr(dev, &sh.diag));
  } else {
    ICP_TRY(tile_counter(st, &sh.tile_counter));
  }
  if (epi == EPI_STORE) {
    if (!a_mn && !b_mn) return launch_umma<false, false, EPI_STORE>(ta, tb, tb2, tc, sh, ep, st, cg, wide);
    if (!a_mn && b_mn) return launch_umma<false, true, EPI_STORE>(ta, tb, tb2, tc, sh, ep, st, cg, wide);
    if (a_mn && !b_mn) return launch_umma<true, false, EPI_STORE>(ta, tb, tb2, tc, sh, ep, st, cg, wide);
    return launch_umma<true, true, EPI_STORE>(ta, tb, tb2, tc, sh, ep, st, cg, wide);
  }
  if (a_mn) return fail(ICEPOP_EINVAL, "fused epilogues need a K-major hidden operand");
  switch (epi) {
    case EPI_LSE:
      return b_mn ? launch_umma<false, true, EPI_LSE>(ta, tb, tb2, tc, sh, ep, st, cg, wide)
                  : launch_umma<false, false, EPI_LSE>(ta, tb, tb2, tc, sh, ep, st, cg, wide);
    case EPI_DZ:
      return b_mn ? launch_umma<false, true, EPI_DZ>(ta, tb, tb2, tc, sh, ep, st, cg)
                  : launch_umma<false, false, EPI_DZ>(ta, tb, tb2, tc, sh, ep, st, cg);
    case EPI_LSE_REF:
      return b_mn ? launch_umma<false, true, EPI_LSE_REF>(ta, tb, tb2, tc, sh, ep, st, cg)
                  : launch_umma<false, false, EPI_LSE_REF>(ta, tb, tb2, tc, sh, ep, st, cg);
    case EPI_DZ_REF:
      return b_mn ? launch_umma<false, true, EPI_DZ_REF>(ta, tb, tb2, tc, sh, ep, st, cg)
                  : launch_umma<false, false, EPI_DZ_REF>(ta, tb, tb2, tc, sh, ep, st, cg);
    default:
      return fail(ICEPOP_EINVAL, "unknown epilogue %d", epi);
  }
}

// ------------------------------------------------------------------ validation helpers
int check_config(const icepop_config* c) {
  if (!c) return fail(ICEPOP_EINVAL, "null config");
  // MaskingBounds.__post_init__ (objective.py:54-56), ObjectiveConfig (objective.py:74-82)
  if (!(0.0 < c->alpha && c->alpha <= 1.0 && 1.0 <= c->beta))
    return fail(ICEPOP_EINVAL, "bounds must satisfy 0 < alpha <= 1 <= beta, got [%g, %g]", c->alpha, c->beta);
  if (!(0.0 < c->clip_eps && c->clip_eps < 1.0)) return fail(ICEPOP_EINVAL, "clip_eps must be in (0, 1)");
  if (!(c->kl_coeff >= 0.0)) return fail(ICEPOP_EINVAL, "kl_coeff must be nonnegative");
  if (!(c->tis_cap > 0.0)) return fail(ICEPOP_EINVAL, "tis_cap must be positive");
  if (!(c->temperature > 0.0)) return fail(ICEPOP_EINVAL, "temperature must be positive");
  if (c->algo < 0 || c->algo > 2) return fail(ICEPOP_EINVAL, "unknown algo %d", c->algo);
  return ICEPOP_OK;
}

int check_shape(const icepop_shape* s, bool bf16) {
  if (!s) return fail(ICEPOP_EINVAL, "null shape");
  if (s->n_tokens < 0 || s->token_offset < 0) return fail(ICEPOP_EINVAL, "negative token range");
  if (s->hidden <= 0 || s->vocab <= 0) return fail(ICEPOP_EINVAL, "hidden and vocab must be positive");
  if (s->n_seqs <= 0 || s->n_groups <= 0)
    return fail(ICEPOP_EINVAL, "objective needs at least one prompt group");
  if (s->weight_layout != ICEPOP_W_DV && s->weight_layout != ICEPOP_W_VD)
    return fail(ICEPOP_EINVAL, "unknown weight layout");
  if (bf16 && (s->hidden % 8 != 0 || s->vocab % 8 != 0))
    return fail(ICEPOP_EINVAL, "bf16 path needs hidden and vocab multiples of 8 (got %lld, %lld)",
                (long long)s->hidden, (long long)s->vocab);
  return ICEPOP_OK;
}

// Per-sequence advantages: given, or K0 from rewards (objective.py:153-159).
int prepare_advantages(const icepop_shape* s, const icepop_batch* b, double* ws_adv, const double** adv,
                       cudaStream_t st) {
  if (b->advantages) {
    *adv = b->advantages;
    return ICEPOP_OK;
  }
  if (!b->rewards) return fail(ICEPOP_EINVAL, "either advantages or rewards must be given");
  const int nb = (s->n_groups + 127) / 128;
  k0_group_advantages<<<nb, 128, 0, st>>>(b->rewards, b->group_offsets, s->n_groups, ws_adv);
  ICP_CUDA(cudaGetLastError());
  *adv = ws_adv;
  return ICEPOP_OK;
}

int token_grid(int64_t n) {
  int64_t g = (n + TOK_THREADS - 1) / TOK_THREADS;
  g = std::min<int64_t>(g, (int64_t)num_sms() * 8);
  return (int)std::max<int64_t>(g, 1);
}

void fill_token_args(TokenArgs& a, const icepop_shape* s, const icepop_config* c, const icepop_batch* b,
                     const double* adv) {
  memset(&a, 0, sizeof(a));
  a.n_tokens = s->n_tokens;
  a.token_offset = s->token_offset;
  a.n_seqs = s->n_seqs;
  a.n_groups = s->n_groups;
  a.tokens = b->tokens;
  a.lp_old = b->lp_train_old;
  a.lp_inf = b->lp_infer_old;
  a.cu_seqlens = b->cu_seqlens;
  a.group_offsets = b->group_offsets;
  a.adv = adv;
  a.calib_in = b->calib;
  a.alpha = c->alpha;
  a.beta = c->beta;
  a.clip_eps = c->clip_eps;
  a.tis_cap = c->tis_cap;
  a.temperature = c->temperature;
  a.kl_coeff = c->kl_coeff;
  a.algo = c->algo;
}

__global__ void k_check_tokens(const int32_t* tokens, int64_t n, int64_t V, unsigned* err) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int y = tokens[t];
    if (y < 0 || y >= V) atomicOr(err, ERR_BAD_TOKEN);
  }
}

__global__ void k_merge_err(const unsigned* err, double* stats) {
  const unsigned e = (unsigned)stats[ICEPOP_STAT_ERRORS] | *err;
  stats[ICEPOP_STAT_ERRORS] = (double)e;
}

__global__ void k_scale_f64(double* z, int64_t n, double temperature) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z[i] = z[i] / temperature;
}

int gemm_f64(const double* A, int64_t sam, int64_t sak, const double* B, int64_t sbk, int64_t sbn, double* C,
             int64_t ldc, int64_t M, int64_t N, int64_t K, int accumulate, cudaStream_t st) {
  if (M <= 0 || N <= 0) return ICEPOP_OK;
  if ((M + F64_TM - 1) / F64_TM > 65535) return fail(ICEPOP_EINVAL, "fp64 validation path: too many rows");
  dim3 grid((unsigned)((N + F64_TN - 1) / F64_TN), (unsigned)((M + F64_TM - 1) / F64_TM));
  k_gemm_f64<<<grid, 256, 0, st>>>(A, sam, sak, B, sbk, sbn, C, ldc, (int)M, (int)N, (int)K, accumulate);
  ICP_CUDA(cudaGetLastError());
  return ICEPOP_OK;
}

// Z[N,V] = H[N,d] . W  (W in layout)
int logits_f64(const icepop_shape* s, const double* H, const double* W, double* Z, cudaStream_t st) {
  const int64_t N = s->n_tokens, d = s->hidden, V = s->vocab;
  if (s->weight_layout == ICEPOP_W_DV) return gemm_f64(H, d, 1, W, V, 1, Z, V, N, V, d, 0, st);
  return gemm_f64(H, d, 1, W, 1, d, Z, V, N, V, d, 0, st);
}

struct BF16Workspace {
  float* part;
  float* ztok;
  double* adv;
  double* block_stats;
  unsigned* err;
  // backward, active-row compaction (skip mode)
  int32_t* idx;
  int32_t* block_counts;
  int32_t* block_offsets;
  int32_t* n_active;
  __nv_bfloat16* hid_act;
  int32_t* tok_act;
  float* lse_act;
  float* coeff_act;
  double* lp_act;
  __nv_bfloat16* dz;
  __nv_bfloat16* hid_t;  // [d, ldt] the dZ chunk's hidden rows transposed (K5's K-major operand)
  int64_t ldt;
  int64_t chunk;
  size_t bytes;
};

// Rows with a zero gradient coefficient are skipped in the backward unless
// ICEPOP_SKIP_INACTIVE=0.
int g_skip_inactive = -1;

bool skip_inactive() {
  if (g_skip_inactive < 0) {
    const char* e = getenv("ICEPOP_SKIP_INACTIVE");
    g_skip_inactive = (e && atoi(e) == 0) ? 0 : 1;
  }
  return g_skip_inactive == 1;
}

// Forward part (partials, stats) is always carved; `bwd` adds the compaction buffers and
// `chunk` rows of bf16 dZ. `ref`: KL-to-ref partials (6 rows per 128-column vocab tile).
BF16Workspace carve_bf16(const icepop_shape* s, void* base, int64_t chunk, bool bwd = false, bool ref = false) {
  Carver c(base);
  BF16Workspace w;
  memset(&w, 0, sizeof(w));
  const int64_t n = std::max<int64_t>(s->n_tokens, 1);
  if (!bwd) {  // the backward reads none of the forward's scratch
    // K1: two partials per run (k1_parts); KL: one per 128-column tile
    const int64_t n_parts = ref ? (s->vocab + bn_of(EPI_LSE_REF) - 1) / bn_of(EPI_LSE_REF) : k1_parts(n, s->vocab, s->hidden);
    w.part = c.take<float>((size_t)n_parts * (ref ? 6 : 3) * n);
    w.ztok = c.take<float>((size_t)n);
    w.adv = c.take<double>((size_t)s->n_seqs);
    w.block_stats = c.take<double>((size_t)num_sms() * 8 * ICEPOP_NSTATS);
    w.err = c.take<unsigned>(4);
  }
  if (bwd && skip_inactive()) {
    const int64_t nb = (n + COMPACT_BLOCK - 1) / COMPACT_BLOCK;
    w.idx = c.take<int32_t>((size_t)n);
    w.block_counts = c.take<int32_t>((size_t)nb);
    w.block_offsets = c.take<int32_t>((size_t)nb);
    w.n_active = c.take<int32_t>(4);
    w.hid_act = c.take<__nv_bfloat16>((size_t)n * s->hidden);
    w.tok_act = c.take<int32_t>((size_t)n);
    w.lse_act = c.take<float>((size_t)n);
    w.coeff_act = c.take<float>((size_t)n);
    w.lp_act = c.take<double>((size_t)n);
  }
  w.dz = c.take<__nv_bfloat16>((size_t)chunk * (size_t)s->vocab);
  if (bwd && chunk > 0) {
    w.ldt = (chunk + 63) / 64 * 64;
    w.hid_t = c.take<__nv_bfloat16>((size_t)w.ldt * s->hidden);
  }
  w.chunk = chunk;
  w.bytes = align_up(c.off, 256);
  return w;
}

// Stored-probabilities backward workspace: block lists of the block-sparse K4/K5
// (k_block_lists) and the row-scaled GEMM inputs (k_sp_prep, the one-hot scatter's sort).
struct SparseWorkspace {
  int32_t* flags;   // [nb] active 64-token blocks
  int32_t* kb_map;  // [nb]
  int32_t* mt_map;  // [nb]
  int32_t* cnt;     // [2]: active blocks, active m-tiles
  float* rscale;    // [n] s_t
  float* ohc;       // [n] c_t
  uint8_t* exc;     // [n] exception rows (dZ formed in place)
  __nv_bfloat16* hid_t;  // [d, ldt] s_t H[t] transposed (k_sp_prep), ldt = n rounded up to 64
  int64_t ldt;
  int32_t* keys;    // [n] tokens sorted
  int32_t* iota;    // [n]
  int32_t* vals;    // [n] token indices sorted by token
  void* sort_tmp;
  size_t sort_bytes;
  size_t bytes;
};

int sort_key_bits(int64_t vocab) {
  int b = 1;
  while ((int64_t(1) << b) < vocab) ++b;
  return b;
}

SparseWorkspace carve_sparse(const icepop_shape* s, void* base) {
  Carver c(base);
  SparseWorkspace w;
  memset(&w, 0, sizeof(w));
  const int64_t n = std::max<int64_t>(s->n_tokens, 1);
  const int64_t nb = (n + 63) / 64;
  w.flags = c.take<int32_t>((size_t)nb);
  w.kb_map = c.take<int32_t>((size_t)nb);
  w.mt_map = c.take<int32_t>((size_t)nb);
  w.cnt = c.take<int32_t>(4);
  w.rscale = c.take<float>((size_t)n);
  w.ohc = c.take<float>((size_t)n);
  w.exc = c.take<uint8_t>((size_t)n);
  w.ldt = (n + 63) / 64 * 64;
  w.hid_t = c.take<__nv_bfloat16>((size_t)w.ldt * s->hidden);
  w.keys = c.take<int32_t>((size_t)n);
  w.iota = c.take<int32_t>((size_t)n);
  w.vals = c.take<int32_t>((size_t)n);
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, (const int32_t*)nullptr, (int32_t*)nullptr, (const int32_t*)nullptr,
                                  (int32_t*)nullptr, (int)n, 0, sort_key_bits(s->vocab));
  w.sort_bytes = std::max<size_t>(tb, 1);
  w.sort_tmp = c.take<uint8_t>(w.sort_bytes);
  w.bytes = align_up(c.off, 256);
  return w;
}

int64_t fwd_part_bytes(const icepop_shape* s, bool ref) {
  BF16Workspace w = carve_bf16(s, nullptr, 0, false, ref);
  return (int64_t)w.bytes;
}

// K3 for `rows` rows of hidden starting at h (saved-tensor pointers already offset). With
// `weight_ref` and saved->kl set it is the dual-accumulator KL variant (gamma > 0).
int launch_dz(const icepop_shape* shape, double temperature, const void* h, const void* weight,
              const void* weight_ref, const icepop_saved& sv, double grad_scale, __nv_bfloat16* dz, int64_t ldz,
              int64_t rows, cudaStream_t st, Extent ext = Extent()) {
  const int64_t d = shape->hidden, V = shape->vocab;
  const bool dv = shape->weight_layout == ICEPOP_W_DV;
  const bool ref = weight_ref && sv.kl && sv.lse_ref && sv.kl_w;
  EpiParams ep;
  memset(&ep, 0, sizeof(ep));
  ep.scale_log2 = (float)(1.4426950408889634 / temperature);
  ep.inv_t = (float)(1.0 / temperature);
  ep.targets = sv.tokens;
  ep.lse = sv.lse;
  ep.coeff = sv.coeff;
  ep.lp_cur = sv.lp_cur;
  ep.lse_ref = sv.lse_ref;
  ep.kl = sv.kl;
  ep.kl_w = sv.kl_w;
  ep.coeff_scale = (float)grad_scale;
  ep.dz = dz;
  ep.ldz = ldz;
  ep.vec_ok = (ldz % 8 == 0) && ((reinterpret_cast<uintptr_t>(dz) & 15u) == 0);
  ep.zero_rows_to = (int32_t)rows;
  return run_umma(ref ? EPI_DZ_REF : EPI_DZ, h, d, false, weight, dv ? V : d, dv, rows, V, d, ep, st, ext,
                  ref ? weight_ref : nullptr);
}

icepop_saved offset_saved(const icepop_saved& s, int64_t o) {
  icepop_saved r = s;
  r.tokens = s.tokens + o;
  r.lse = s.lse + o;
  r.coeff = s.coeff + o;
  if (s.lp_cur) r.lp_cur = s.lp_cur + o;
  if (s.lse_ref) r.lse_ref = s.lse_ref + o;
  if (s.kl) r.kl = s.kl + o;
  if (s.kl_w) r.kl_w = s.kl_w + o;
  return r;
}

// K2 (merge of K1's partials + the IcePop epilogue) and the fixed-order stats reduction, from
// the forward workspace `w` (partials, ztok, token-check error word).
int run_k2(const icepop_shape* shape, const icepop_config* cfg, const icepop_batch* batch, const icepop_fwd_out* out,
           const BF16Workspace& w, bool ref, const double* adv, cudaStream_t st) {
  const int64_t N = shape->n_tokens, d = shape->hidden, V = shape->vocab;
  TokenArgs a;
  fill_token_args(a, shape, cfg, batch, adv);
  if (!ref) a.kl_coeff = 0.0;  // no reference policy: kl_t = 0 (objective.py:254)
  a.part = w.part;
  a.n_parts = (int32_t)(ref ? (V + bn_of(EPI_LSE_REF) - 1) / bn_of(EPI_LSE_REF) : k1_parts(N, V, d));
  a.part_cols = ref ? bn_of(EPI_LSE_REF) : k1_part_cols(N, V, d);
  a.kl_f = ref ? out->kl : nullptr;
  a.lse_ref_f = ref ? out->lse_ref : nullptr;
  a.kl_w_f = ref ? out->kl_w : nullptr;
  a.ztok = w.ztok;
  a.lse_f = out->lse;
  a.lp_cur = out->lp_cur;
  a.entropy_f = out->entropy;
  a.kept = out->kept;
  a.calib = out->calib;
  a.surrogate = out->surrogate;
  a.coeff_f = out->coeff;
  a.block_stats = w.block_stats;
  const int grid = token_grid(N);
  if (ref) k2_icepop_tokens<3><<<grid, TOK_THREADS, 0, st>>>(a);
  else k2_icepop_tokens<0><<<grid, TOK_THREADS, 0, st>>>(a);
  ICP_CUDA(cudaGetLastError());
  k_finalize_stats<<<1, 32 * ICEPOP_NSTATS, 0, st>>>(w.block_stats, grid, out->stats);
  k_merge_err<<<1, 1, 0, st>>>(w.err, out->stats);
  ICP_CUDA(cudaGetLastError());
  return ICEPOP_OK;
}

}  // namespace

// =====================================================================================
extern "C" {

int icepop_abi_version(void) { return ICEPOP_ABI_VERSION; }

const char* icepop_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"

static int preload_kernels();

extern "C" {

int icepop_device_check(int device) {
  cudaDeviceProp p;
  cudaError_t e = cudaGetDeviceProperties(&p, device);
  if (e != cudaSuccess) return fail(ICEPOP_ECUDA, "cudaGetDeviceProperties: %s", cudaGetErrorString(e));
  if (p.major != 10 || p.minor != 0)
    return fail(ICEPOP_EARCH, "libicepop_b200 is built for sm_100a; device %d is sm_%d%d", device, p.major, p.minor);
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, umma_gemm_kernel<BN_, false, false, EPI_LSE, 2>);
  if (e != cudaSuccess) return fail(ICEPOP_EARCH, "sm_100a kernels not loadable: %s", cudaGetErrorString(e));
  int cur = 0;
  ICP_CUDA(cudaGetDevice(&cur));
  ICP_CUDA(cudaSetDevice(device));
  int rc = ensure_pool(device);  // scheduler counters: allocated here, never inside a capture
  if (rc == ICEPOP_OK) rc = preload_kernels();
  cudaSetDevice(cur);
  return rc;
}

int icepop_group_advantages(const double* rewards, const int32_t* group_offsets, int32_t n_groups, int32_t n_seqs,
                            double* advantages, void* stream) {
  if (!rewards || !group_offsets || !advantages || n_groups <= 0 || n_seqs <= 0)
    return fail(ICEPOP_EINVAL, "invalid group_advantages arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k0_group_advantages<<<(n_groups + 127) / 128, 128, 0, st>>>(rewards, group_offsets, n_groups, advantages);
  ICP_CUDA(cudaGetLastError());
  return ICEPOP_OK;
}

int icepop_workspace_bytes(const icepop_shape* shape, int64_t max_chunk_tokens, int32_t with_ref,
                           size_t* fwd_bytes, size_t* bwd_bytes) {
  ICP_TRY(check_shape(shape, true));
  int64_t chunk = shape->n_tokens;
  if (max_chunk_tokens > 0) chunk = std::min<int64_t>(chunk, max_chunk_tokens);
  chunk = std::max<int64_t>(chunk, 1);
  if (fwd_bytes) *fwd_bytes = (size_t)fwd_part_bytes(shape, with_ref != 0);
  if (bwd_bytes)  // max_chunk_tokens < 0: the stored-probabilities backward (block lists only)
    *bwd_bytes = max_chunk_tokens < 0 ? carve_sparse(shape, nullptr).bytes : carve_bf16(shape, nullptr, chunk, true).bytes;
  return ICEPOP_OK;
}

int icepop_fwd_bf16(const icepop_shape* shape, const icepop_config* cfg, const void* hidden, const void* weight,
                    const void* weight_ref, const icepop_batch* batch, const icepop_fwd_out* out, void* workspace,
                    size_t workspace_bytes, void* stream) {
  ICP_TRY(check_shape(shape, true));
  ICP_TRY(check_config(cfg));
  if (!batch || !out || !out->stats) return fail(ICEPOP_EINVAL, "null batch/out/stats");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool ref = weight_ref != nullptr;
  BF16Workspace w = carve_bf16(shape, workspace, 0, false, ref);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(ICEPOP_EINVAL, "forward workspace too small: need %zu bytes", w.bytes);
  const int64_t N = shape->n_tokens, d = shape->hidden, V = shape->vocab;
  if (out->probs) {
    // with gamma > 0 the backward needs the KL term's gradient, which the recompute forms
    if (ref && cfg->kl_coeff > 0.0)
      return fail(ICEPOP_EINVAL, "stored probabilities with weight_ref need kl_coeff == 0 (the KL term then "
                                 "enters J only)");
    if (!out->tile_max) return fail(ICEPOP_EINVAL, "stored probabilities need out->tile_max");
    if (V % 8 != 0) return fail(ICEPOP_EINVAL, "stored probabilities need vocab %% 8 == 0");
    if (((reinterpret_cast<uintptr_t>(out->probs) | reinterpret_cast<uintptr_t>(out->tile_max)) & 15u) != 0)
      return fail(ICEPOP_EINVAL, "out->probs and out->tile_max must be 16-byte aligned");
  }
  const double* adv = nullptr;
  ICP_TRY(prepare_advantages(shape, batch, w.adv, &adv, st));
  ICP_CUDA(cudaMemsetAsync(w.err, 0, sizeof(unsigned), st));
  if (N > 0) {
    k_check_tokens<<<token_grid(N), TOK_THREADS, 0, st>>>(batch->tokens, N, V, w.err);
    ICP_CUDA(cudaGetLastError());
    // K1: fused lm_head GEMM + online softmax statistics (logits stay in TMEM)
    EpiParams ep;
    memset(&ep, 0, sizeof(ep));
    ep.scale_log2 = (float)(1.4426950408889634 / cfg->temperature);
    ep.inv_t = (float)(1.0 / cfg->temperature);
    ep.targets = batch->tokens;
    ep.part = w.part;
    ep.ztok = w.ztok;
    ep.probs = static_cast<__nv_bfloat16*>(out->probs);
    ep.tile_max = out->tile_max;
    ep.tm_ld = (int32_t)(4 * ((V + BN_ - 1) / BN_));  // four 64-column slab maxima per 256-column tile
    const bool b_mn = shape->weight_layout == ICEPOP_W_DV;
    ICP_TRY(run_umma(ref ? EPI_LSE_REF : EPI_LSE, hidden, d, false, weight, b_mn ? V : d, b_mn, N, V, d, ep, st,
                     Extent(), ref ? weight_ref : nullptr));
  }
  return run_k2(shape, cfg, batch, out, w, ref, adv, st);
}

int icepop_fwd_epilogue_bf16(const icepop_shape* shape, const icepop_config* cfg, const icepop_batch* batch,
                             int32_t with_ref, const icepop_fwd_out* out, void* workspace, size_t workspace_bytes,
                             void* stream) {
  ICP_TRY(check_shape(shape, true));
  ICP_TRY(check_config(cfg));
  if (!batch || !out || !out->stats) return fail(ICEPOP_EINVAL, "null batch/out/stats");
  const bool ref = with_ref != 0;
  BF16Workspace w = carve_bf16(shape, workspace, 0, false, ref);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(ICEPOP_EINVAL, "forward workspace too small: need %zu bytes", w.bytes);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const double* adv = nullptr;
  ICP_TRY(prepare_advantages(shape, batch, w.adv, &adv, st));
  return run_k2(shape, cfg, batch, out, w, ref, adv, st);
}

int icepop_fwd_onpolicy(const icepop_shape* shape, const icepop_config* cfg, const icepop_batch* batch,
                        const float* lse_old, const float* entropy_old, const icepop_fwd_out* out, void* workspace,
                        size_t workspace_bytes, void* stream) {
  ICP_TRY(check_shape(shape, false));
  ICP_TRY(check_config(cfg));
  if (!batch || !out || !out->stats || !lse_old) return fail(ICEPOP_EINVAL, "null batch/out/stats/lse_old");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  BF16Workspace w = carve_bf16(shape, workspace, 0, false, false);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(ICEPOP_EINVAL, "forward workspace too small: need %zu bytes", w.bytes);
  const int64_t N = shape->n_tokens, V = shape->vocab;
  const double* adv = nullptr;
  ICP_TRY(prepare_advantages(shape, batch, w.adv, &adv, st));
  ICP_CUDA(cudaMemsetAsync(w.err, 0, sizeof(unsigned), st));
  if (N > 0) {
    k_check_tokens<<<token_grid(N), TOK_THREADS, 0, st>>>(batch->tokens, N, V, w.err);
    ICP_CUDA(cudaGetLastError());
  }
  TokenArgs a;
  fill_token_args(a, shape, cfg, batch, adv);
  a.kl_coeff = 0.0;
  a.lse_in = lse_old;
  a.entropy_in_f = entropy_old;
  a.lse_f = out->lse;
  a.lp_cur = out->lp_cur;
  a.entropy_f = out->entropy;
  a.kept = out->kept;
  a.calib = out->calib;
  a.surrogate = out->surrogate;
  a.coeff_f = out->coeff;
  a.block_stats = w.block_stats;
  const int grid = token_grid(N);
  k2_icepop_tokens<2><<<grid, TOK_THREADS, 0, st>>>(a);
  ICP_CUDA(cudaGetLastError());
  k_finalize_stats<<<1, 32 * ICEPOP_NSTATS, 0, st>>>(w.block_stats, grid, out->stats);
  k_merge_err<<<1, 1, 0, st>>>(w.err, out->stats);
  ICP_CUDA(cudaGetLastError());
  return ICEPOP_OK;
}

__global__ void k_logprob_finish(const float* part, int n_parts, int32_t part_cols, const int32_t* tokens,
                                 const float* ztok, int64_t n, float* lse, double* lp, float* entropy) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const float my = __ldg(part + token_part(__ldg(tokens + t), part_cols, n_parts) * 3 * n + t);
    PartMerge pm;  // one pass with a running maximum (k2_icepop_tokens)
    merge_partials<3>(pm, part, n_parts, n, t);
    float l, e;
    double lpv;
    pm.finish(ztok[t], my, l, lpv, e);
    if (lse) lse[t] = l;
    if (lp) lp[t] = lpv;
    if (entropy) entropy[t] = e;
  }
}

int icepop_logprob_bf16(const icepop_shape* shape, double temperature, const void* hidden, const void* weight,
                        const int32_t* tokens, float* lse, double* lp, float* entropy, void* workspace,
                        size_t workspace_bytes, void* stream) {
  ICP_TRY(check_shape(shape, true));
  if (!(temperature > 0.0)) return fail(ICEPOP_EINVAL, "temperature must be positive");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  BF16Workspace w = carve_bf16(shape, workspace, 0, false, false);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(ICEPOP_EINVAL, "workspace too small: need %zu bytes", w.bytes);
  const int64_t N = shape->n_tokens, d = shape->hidden, V = shape->vocab;
  if (N == 0) return ICEPOP_OK;
  EpiParams ep;
  memset(&ep, 0, sizeof(ep));
  ep.scale_log2 = (float)(1.4426950408889634 / temperature);
  ep.inv_t = (float)(1.0 / temperature);
  ep.targets = tokens;
  ep.part = w.part;
  ep.ztok = w.ztok;
  const bool b_mn = shape->weight_layout == ICEPOP_W_DV;
  ICP_TRY(run_umma(EPI_LSE, hidden, d, false, weight, b_mn ? V : d, b_mn, N, V, d, ep, st));
  k_logprob_finish<<<token_grid(N), TOK_THREADS, 0, st>>>(w.part, (int)k1_parts(N, V, d), k1_part_cols(N, V, d),
                                                          tokens, w.ztok, N, lse, lp, entropy);
  ICP_CUDA(cudaGetLastError());
  return ICEPOP_OK;
}

}  // extern "C"

// Backward implementation. With `rs`, grad_weight is this rank's LOCAL scratch for earlier
// token chunks (may be null with a single chunk) and the last chunk's K5 epilogue stores
// every dW row into its owner's peer slot (fused reduce-scatter over NVLink).
static int bwd_impl(const icepop_shape* shape, const icepop_config* cfg, const void* hidden, const void* weight,
                    const void* weight_ref, const icepop_saved* saved, double grad_scale, void* grad_hidden,
                    int32_t grad_hidden_f32, float* grad_weight, int32_t accumulate, void* workspace,
                    size_t workspace_bytes, void* stream, const icepop_rs_target* rs) {
  ICP_TRY(check_shape(shape, true));
  ICP_TRY(check_config(cfg));
  if (!saved || !saved->tokens || !saved->lse || !saved->coeff) return fail(ICEPOP_EINVAL, "null saved tensors");
  // the KL term only enters the gradient when gamma > 0 (objective.py:259)
  const bool kl_grad = weight_ref && cfg->kl_coeff > 0.0;
  if (kl_grad && (!saved->kl || !saved->lse_ref || !saved->kl_w))
    return fail(ICEPOP_EINVAL, "the KL gradient needs saved kl, lse_ref and kl_w");
  icepop_saved sv = *saved;
  if (!kl_grad) sv.kl = sv.lse_ref = sv.kl_w = nullptr;
  const int32_t* tokens = sv.tokens;
  const float* lse = sv.lse;
  const float* coeff = sv.coeff;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t N = shape->n_tokens, d = shape->hidden, V = shape->vocab;
  const bool dv = shape->weight_layout == ICEPOP_W_DV;
  if (N == 0 && rs) return fail(ICEPOP_EINVAL, "fused reduce-scatter needs at least one local token");
  if (N == 0) {
    if (grad_weight && !accumulate) ICP_CUDA(cudaMemsetAsync(grad_weight, 0, sizeof(float) * d * V, st));
    return ICEPOP_OK;
  }
  // stored-probabilities mode: dZ is formed in place over saved->probs (one chunk, all rows)
  const bool sp = sv.probs != nullptr;
  if (sp) {
    if (kl_grad) return fail(ICEPOP_EINVAL, "stored probabilities carry no KL term: gamma > 0 needs recompute mode");
    if (!sv.tile_max) return fail(ICEPOP_EINVAL, "saved->probs needs saved->tile_max");
    if (V % 8 != 0 || (reinterpret_cast<uintptr_t>(sv.probs) & 15u) != 0)
      return fail(ICEPOP_EINVAL, "saved->probs needs vocab %% 8 == 0 and 16-byte alignment");
    if (!sv.lp_cur) return fail(ICEPOP_EINVAL, "saved->probs needs saved->lp_cur (the sampled token's exact term)");
  }
  // chunk = as many dZ rows as the workspace holds (all rows, or a multiple of 128)
  bool skip = skip_inactive() && !kl_grad;  // with gamma > 0 every row has a KL gradient
  int64_t chunk = N;
  BF16Workspace w;
  memset(&w, 0, sizeof(w));
  // stored probabilities: dZ in place over all rows (zero-coefficient rows become zero rows),
  // then K4/K5 skip the 64-token blocks / 256-token tiles without any active row when the
  // workspace holds the block lists (block-sparse GEMMs; no data moves)
  // With its workspace the stored-probabilities backward is row-scaled: no dZ pass except for
  // exception rows (k_sp_prep), K4 scales rows and adds c W[y], K5 reads s H, and the one-hot
  // part of dW is a deterministic scatter. Without it: dZ in place over every row.
  bool sparse = false, scaled = false;
  SparseWorkspace sw;
  memset(&sw, 0, sizeof(sw));
  if (sp) {
    if (workspace && workspace_bytes >= carve_sparse(shape, nullptr).bytes) {
      sw = carve_sparse(shape, workspace);
      scaled = true;  // (with the fused reduce-scatter the one-hot part goes straight to the slots)
      sparse = skip;
    }
    skip = false;
  } else {
    const int64_t min_rows = std::min<int64_t>(N, BM);
    const size_t need_min = carve_bf16(shape, nullptr, min_rows, true).bytes;
    if (!workspace || workspace_bytes < need_min)
      return fail(ICEPOP_EINVAL, "backward workspace too small: need >= %zu bytes", need_min);
    const size_t fixed = carve_bf16(shape, nullptr, 0, true).bytes;
    chunk = (int64_t)((workspace_bytes - fixed) / ((size_t)(V + d) * 2));  // dZ row + transposed H row
    if (chunk >= N) {
      chunk = N;
    } else {
      chunk = std::max<int64_t>(chunk / BM * BM, BM);
    }
    while (chunk > min_rows && carve_bf16(shape, nullptr, chunk, true).bytes > workspace_bytes) chunk -= BM;
    w = carve_bf16(shape, workspace, chunk, true);
    if (w.bytes > workspace_bytes) return fail(ICEPOP_EINVAL, "backward workspace carve overflow");
  }
  __nv_bfloat16* dzb = sp ? static_cast<__nv_bfloat16*>(sv.probs) : w.dz;

  const void* hsrc = hidden;
  const int32_t* tok_src = tokens;
  const float* lse_src = lse;
  const float* coeff_src = coeff;
  const size_t gh_esz = grad_hidden_f32 ? 4 : 2;
  if (skip) {
    // compact the rows with coeff != 0 (device-side count: no host sync)
    const int nb = (int)((N + COMPACT_BLOCK - 1) / COMPACT_BLOCK);
    k_active_count<<<nb, COMPACT_BLOCK, 0, st>>>(coeff, N, w.block_counts);
    k_active_scan<<<1, std::min(1024, nb), 0, st>>>(w.block_counts, nb, w.block_offsets, w.n_active);
    k_active_scatter<<<nb, COMPACT_BLOCK, 0, st>>>(coeff, N, w.block_offsets, w.idx);
    const int64_t d8 = d / 8;
    const int gg = (int)std::min<int64_t>((N * d8 + 255) / 256, (int64_t)num_sms() * 16);
    k_gather_active<<<gg, 256, 0, st>>>(w.idx, w.n_active, reinterpret_cast<const uint4*>(hidden), d8, tokens, lse,
                                        coeff, reinterpret_cast<uint4*>(w.hid_act), w.tok_act, w.lse_act,
                                        w.coeff_act, sv.lp_cur, w.lp_act, N);
    ICP_CUDA(cudaGetLastError());
    if (grad_hidden) ICP_CUDA(cudaMemsetAsync(grad_hidden, 0, (size_t)N * d * gh_esz, st));
    hsrc = w.hid_act;
    tok_src = w.tok_act;
    lse_src = w.lse_act;
    coeff_src = w.coeff_act;
  }

  const int64_t n_chunks = (N + chunk - 1) / chunk;
  if (rs && n_chunks > 1 && !grad_weight)
    return fail(ICEPOP_EINVAL, "fused reduce-scatter over several dZ chunks needs a local grad_weight scratch");
  for (int64_t c0 = 0; c0 < N; c0 += chunk) {
    const int64_t nc = std::min<int64_t>(chunk, N - c0);
    const bool last = c0 + chunk >= N;
    const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(hsrc) + c0 * d;
    Extent ext_m, ext_k;
    if (skip) {
      ext_m.dev = w.n_active;
      ext_m.base = (int32_t)c0;
      ext_m.dim = 1;
      ext_k = ext_m;
      ext_k.dim = 2;
    }
    // K3: recompute logits, dZ chunk (bf16)
    icepop_saved cs = offset_saved(sv, c0);
    if (skip) {
      cs.tokens = tok_src + c0;
      cs.lse = lse_src + c0;
      cs.coeff = coeff_src + c0;
      cs.lp_cur = sv.lp_cur ? w.lp_act + c0 : nullptr;
    }
    if (sp) {
      const int32_t tm_ld = (int32_t)(4 * ((V + BN_ - 1) / BN_));
      if (sparse) {
        const int64_t nb = (nc + 63) / 64;
        k_block_flags<<<(int)((nb * 32 + 255) / 256), 256, 0, st>>>(coeff, nc, sw.flags);
        k_block_lists<<<1, BL_THREADS, 0, st>>>(sw.flags, nb, BM * cta_group() / 64, sw.kb_map, sw.mt_map, sw.cnt);
        if (grad_hidden) ICP_CUDA(cudaMemsetAsync(grad_hidden, 0, (size_t)N * d * gh_esz, st));  // skipped tiles
      }
      const int grid = (int)std::min<int64_t>(nc, (int64_t)num_sms() * 8);
      if (scaled) {
        const dim3 pgrid = spp_grid(nc, d);
        k_sp_prep<<<pgrid, SPP_THREADS, 0, st>>>(sv.tile_max, tm_ld, (int32_t)((V + 63) / 64), lse, coeff,
                                                 (float)grad_scale, sv.lp_cur, tokens, dzb, V,
                                                 reinterpret_cast<const uint4*>(hidden), d / 8, sw.rscale, sw.ohc,
                                                 sw.exc, reinterpret_cast<uint4*>(sw.hid_t), sw.ldt, nc);
      }
      k_dz_probs<<<grid, DZP_THREADS, 0, st>>>(reinterpret_cast<uint4*>(dzb), sv.tile_max, tm_ld, lse, coeff,
                                               (float)grad_scale, tokens, nc, V / 8, sv.lp_cur,
                                               scaled ? sw.exc : nullptr);
      ICP_CUDA(cudaGetLastError());
    } else {
      ICP_TRY(launch_dz(shape, cfg->temperature, h, weight, kl_grad ? weight_ref : nullptr, cs, grad_scale, w.dz, V,
                        nc, st, ext_m));
    }
    // K4: grad_hidden = dZ . W^T   (M = nc, N = d, K = V)
    if (grad_hidden) {
      EpiParams eh;
      memset(&eh, 0, sizeof(eh));
      // skip mode scatters compacted row m back to token idx[c0 + m]
      eh.out = skip ? grad_hidden : static_cast<uint8_t*>(grad_hidden) + (size_t)c0 * d * gh_esz;
      eh.row_index = skip ? w.idx + c0 : nullptr;
      eh.ldo = d;
      eh.out_f32 = grad_hidden_f32 ? 1 : 0;
      eh.vec_ok = ((reinterpret_cast<uintptr_t>(eh.out) & 15u) == 0) && (d % 8 == 0);
      if (scaled) {  // dH = s (Q.W) + c W[y]
        eh.row_scale = sw.rscale;
        eh.oh_coef = sw.ohc;
        eh.oh_tok = tokens;
        eh.oh_w = static_cast<const __nv_bfloat16*>(weight);
        eh.oh_sy = dv ? 1 : d;  // W(y, n): [V,d] row y / [d,V] column y
        eh.oh_sn = dv ? V : 1;
      }
      // B operand viewed [N = d, K = V]: W[d,V] is K-major, W[V,d] is MN-major
      Sparse sp4;
      if (sparse) {
        sp4.mt_map = sw.mt_map;
        sp4.mt_cnt = sw.cnt + 1;
      }
      ICP_TRY(run_umma(EPI_STORE, dzb, V, false, weight, dv ? V : d, !dv, nc, d, V, eh, st, ext_m, nullptr, false, sp4));
    }
    // K5: grad_weight (+)= H^T . dZ   (K = nc tokens)
    if (grad_weight || (rs && last)) {
      // row-scaled stored probabilities: dW = Q^T.(s H) + scatter_y(c H); the one-hot part
      // is scattered after K5 into grad_weight, or (fused reduce-scatter) first into the local
      // scratch that K5's epilogue adds to every row it sends
      auto onehot_scatter = [&](float* dw, const icepop_rs_target* to) -> int {
        k_iota<<<(int)std::min<int64_t>((nc + 255) / 256, (int64_t)num_sms() * 8), 256, 0, st>>>(sw.iota, nc);
        size_t tb = sw.sort_bytes;
        ICP_CUDA(cub::DeviceRadixSort::SortPairs(sw.sort_tmp, tb, tokens, sw.keys, sw.iota, sw.vals, (int)nc, 0,
                                                 sort_key_bits(V), st));
        OneHotDst od;
        memset(&od, 0, sizeof(od));
        od.dw = dw;
        od.sy = dv ? 1 : d;
        od.sc = dv ? V : 1;
        od.rows_are_y = dv ? 0 : 1;
        if (to) {
          od.rs_world = to->world;
          od.rs_rank = to->rank;
          od.shard_rows = to->shard_rows;
          od.row_len = dv ? V : d;
          for (int o = 0; o < to->world; ++o) od.slots[o] = to->slots[o];
        }
        k_onehot_scatter<<<(int)std::min<int64_t>(nc, (int64_t)num_sms() * 8), OHS_THREADS, 0, st>>>(
            sw.keys, sw.vals, nc, sw.ohc, reinterpret_cast<const uint4*>(hidden), d / 8, od);
        ICP_CUDA(cudaGetLastError());
        return ICEPOP_OK;
      };
      EpiParams ew;
      memset(&ew, 0, sizeof(ew));
      ew.out = grad_weight;
      ew.out_f32 = 1;
      // with compacted rows the K extent may be empty: K5 still runs its tiles (keep_empty) and
      // stores zeros, so dW needs no memset
      ew.accumulate = (accumulate || c0 > 0) ? 1 : 0;
      if (rs && last) {
        // fused reduce-scatter: store each row (+ this rank's earlier-chunk partial) into the
        // owner's slot over NVLink
        ew.rs_world = rs->world;
        ew.rs_rank = rs->rank;
        ew.rs_shard_rows = rs->shard_rows;
        for (int o = 0; o < rs->world; ++o) ew.rs_slots[o] = rs->slots[o];
        ew.acc_src = (n_chunks > 1) ? grad_weight : nullptr;
        ew.out = nullptr;
        ext_k.dim = skip ? 2 : 0;
      }
      // an empty K extent must still store (zeros, or the local partial to the peers) when
      // nothing else writes the result
      const bool keep_empty = ((skip || sparse) && !ew.accumulate) || (rs && last);
      Sparse sp5;
      if (sparse) {
        sp5.kb_map = sw.kb_map;
        sp5.kb_cnt = sw.cnt;
      }
      const void* ovec = rs && last ? (const void*)rs->slots[0] : (const void*)grad_weight;
      ew.vec_ok = ((reinterpret_cast<uintptr_t>(ovec) & 15u) == 0) && (d % 8 == 0) && (V % 8 == 0);
      // K5's hidden operand K-major (one MN-major operand, not two: profiles/major_ab.py): the
      // row-scaled H' transposed by k_sp_prep, or this chunk's rows transposed here (the
      // recompute backward); H itself (MN-major, [nc, d]) only without either workspace
      if (!scaled && w.hid_t) {
        k_transpose_rows<<<spp_grid(nc, d), SPP_THREADS, 0, st>>>(reinterpret_cast<const uint4*>(h), d / 8,
                                                     reinterpret_cast<uint4*>(w.hid_t), w.ldt, nc);
        ICP_CUDA(cudaGetLastError());
      }
      const bool h_kmajor = scaled || w.hid_t != nullptr;
      const void* hk = scaled ? (const void*)sw.hid_t : (w.hid_t ? (const void*)w.hid_t : (const void*)h);
      const int64_t ldh = scaled ? sw.ldt : (w.hid_t ? w.ldt : d);
      if (dv) {
        ew.ldo = V;  // dW[d,V]: A = H chunk viewed [M=d, K=nc], B = dZ [N=V, K=nc] (MN-major)
        ICP_TRY(run_umma(EPI_STORE, hk, ldh, !h_kmajor, dzb, V, true, d, V, nc, ew, st, ext_k, nullptr, keep_empty,
                         sp5));
      } else {
        ew.ldo = d;  // dW[V,d]: A = dZ viewed [M=V, K=nc] (MN-major), B = H chunk [N=d, K=nc]
        ICP_TRY(run_umma(EPI_STORE, dzb, V, true, hk, ldh, !h_kmajor, V, d, nc, ew, st, ext_k, nullptr, keep_empty,
                         sp5));
      }
      // the one-hot part after K5 stored dW: into grad_weight, or (fused reduce-scatter) straight
      // into the owners' slots, sparse read-modify-writes of the rows the batch's tokens touch
      if (scaled) ICP_TRY(onehot_scatter(grad_weight, rs && last ? rs : nullptr));
    }
  }
  return ICEPOP_OK;
}

extern "C" {

int icepop_bwd_bf16(const icepop_shape* shape, const icepop_config* cfg, const void* hidden, const void* weight,
                    const void* weight_ref, const icepop_saved* saved, double grad_scale, void* grad_hidden,
                    int32_t grad_hidden_f32, float* grad_weight, int32_t accumulate, void* workspace,
                    size_t workspace_bytes, void* stream) {
  return bwd_impl(shape, cfg, hidden, weight, weight_ref, saved, grad_scale, grad_hidden, grad_hidden_f32,
                  grad_weight, accumulate, workspace, workspace_bytes, stream, nullptr);
}

int icepop_bwd_bf16_rs(const icepop_shape* shape, const icepop_config* cfg, const void* hidden, const void* weight,
                       const void* weight_ref, const icepop_saved* saved, double grad_scale, void* grad_hidden,
                       int32_t grad_hidden_f32, const icepop_rs_target* rs, float* grad_weight_scratch,
                       void* workspace, size_t workspace_bytes, void* stream) {
  if (!rs || rs->world < 1 || rs->world > 8 || rs->rank < 0 || rs->rank >= rs->world || rs->shard_rows <= 0)
    return fail(ICEPOP_EINVAL, "invalid reduce-scatter target");
  const int64_t rows = shape ? (shape->weight_layout == ICEPOP_W_DV ? shape->hidden : shape->vocab) : 0;
  if ((int64_t)rs->world * rs->shard_rows < rows) return fail(ICEPOP_EINVAL, "shards do not cover grad_weight");
  for (int o = 0; o < rs->world; ++o)
    if (!rs->slots[o]) return fail(ICEPOP_EINVAL, "null peer slot %d", o);
  return bwd_impl(shape, cfg, hidden, weight, weight_ref, saved, grad_scale, grad_hidden, grad_hidden_f32,
                  grad_weight_scratch, 0, workspace, workspace_bytes, stream, rs);
}

int icepop_rs_fold(const float* slots, int32_t world, int64_t shard_elems, float* out, void* stream) {
  if (!slots || !out || world < 1 || shard_elems < 0 || shard_elems % 4 != 0)
    return fail(ICEPOP_EINVAL, "invalid fold arguments (shard_elems must be a multiple of 4)");
  const int64_t n4 = shard_elems / 4;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n4 + 255) / 256, (int64_t)num_sms() * 8));
  k_rs_fold<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(reinterpret_cast<const float4*>(slots), world, n4,
                                                                 reinterpret_cast<float4*>(out));
  ICP_CUDA(cudaGetLastError());
  return ICEPOP_OK;
}

int icepop_peer_alloc(size_t bytes, void** ptr) {
  if (!ptr) return fail(ICEPOP_EINVAL, "null out pointer");
  ICP_CUDA(cudaMalloc(ptr, std::max<size_t>(bytes, 256)));
  return ICEPOP_OK;
}

int icepop_peer_free(void* ptr) {
  ICP_CUDA(cudaFree(ptr));
  return ICEPOP_OK;
}

int icepop_peer_export(void* ptr, void* handle) {
  if (!ptr || !handle) return fail(ICEPOP_EINVAL, "null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  ICP_CUDA(cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(handle), ptr));
  return ICEPOP_OK;
}

int icepop_peer_import(const void* handle, void** ptr) {
  if (!ptr || !handle) return fail(ICEPOP_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  ICP_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return ICEPOP_OK;
}

int icepop_peer_close(void* ptr) {
  ICP_CUDA(cudaIpcCloseMemHandle(ptr));
  return ICEPOP_OK;
}

int icepop_dz_bf16(const icepop_shape* shape, double temperature, const void* hidden, const void* weight,
                   const void* weight_ref, const icepop_saved* saved, double grad_scale, void* dz, int64_t ldz,
                   void* stream) {
  ICP_TRY(check_shape(shape, true));
  if (!(temperature > 0.0)) return fail(ICEPOP_EINVAL, "temperature must be positive");
  if (!hidden || !weight || !saved || !saved->tokens || !saved->lse || !saved->coeff || !dz)
    return fail(ICEPOP_EINVAL, "null argument");
  if (ldz < shape->vocab) return fail(ICEPOP_EINVAL, "ldz must be >= vocab");
  return launch_dz(shape, temperature, hidden, weight, weight_ref, *saved, grad_scale,
                   static_cast<__nv_bfloat16*>(dz), ldz, shape->n_tokens, static_cast<cudaStream_t>(stream));
}

// ------------------------------------------------------------------ fp64 validation path
int icepop_workspace_bytes_f64(const icepop_shape* shape, int32_t with_ref, size_t* bytes) {
  ICP_TRY(check_shape(shape, false));
  Carver c(nullptr);
  c.take<double>((size_t)shape->n_tokens * shape->vocab);
  if (with_ref) c.take<double>((size_t)shape->n_tokens * shape->vocab);
  c.take<double>((size_t)shape->n_seqs);
  c.take<double>((size_t)num_sms() * 8 * ICEPOP_NSTATS);
  c.take<unsigned>(4);
  c.take<double>((size_t)std::max<int64_t>(shape->n_tokens, 1));
  *bytes = align_up(c.off, 256);
  return ICEPOP_OK;
}

struct F64Workspace {
  double* Z;
  double* Zref;
  double* adv;
  double* block_stats;
  unsigned* err;
  double* kw;
  size_t bytes;
};

static F64Workspace carve_f64(const icepop_shape* s, void* base, bool with_ref) {
  Carver c(base);
  F64Workspace w;
  w.Z = c.take<double>((size_t)s->n_tokens * s->vocab);
  w.Zref = with_ref ? c.take<double>((size_t)s->n_tokens * s->vocab) : nullptr;
  w.adv = c.take<double>((size_t)s->n_seqs);
  w.block_stats = c.take<double>((size_t)num_sms() * 8 * ICEPOP_NSTATS);
  w.err = c.take<unsigned>(4);
  w.kw = c.take<double>((size_t)std::max<int64_t>(s->n_tokens, 1));
  w.bytes = align_up(c.off, 256);
  return w;
}

int icepop_fwd_f64(const icepop_shape* shape, const icepop_config* cfg, const double* hidden, const double* weight,
                   const double* weight_ref, const icepop_batch* batch, const icepop_f64_out* out, void* workspace,
                   size_t workspace_bytes, void* stream) {
  ICP_TRY(check_shape(shape, false));
  ICP_TRY(check_config(cfg));
  if (!batch || !out || !out->stats || !out->lse || !out->lp_cur || !out->entropy)
    return fail(ICEPOP_EINVAL, "null batch/out");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool with_ref = weight_ref != nullptr;
  F64Workspace w = carve_f64(shape, workspace, with_ref);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(ICEPOP_EINVAL, "fp64 workspace too small: need %zu bytes", w.bytes);
  const int64_t N = shape->n_tokens, V = shape->vocab;
  const double* adv = nullptr;
  ICP_TRY(prepare_advantages(shape, batch, w.adv, &adv, st));
  ICP_CUDA(cudaMemsetAsync(w.err, 0, sizeof(unsigned), st));
  if (N > 0) {
    k_check_tokens<<<token_grid(N), TOK_THREADS, 0, st>>>(batch->tokens, N, V, w.err);
    ICP_TRY(logits_f64(shape, hidden, weight, w.Z, st));
    if (with_ref) ICP_TRY(logits_f64(shape, hidden, weight_ref, w.Zref, st));
    k_rowstats_f64<<<(unsigned)N, F64_ROW_THREADS, 0, st>>>(w.Z, w.Zref, V, cfg->temperature, batch->tokens,
                                                            out->lse, out->lp_cur, out->entropy,
                                                            with_ref ? out->kl : nullptr,
                                                            with_ref ? out->lse_ref : nullptr, w.err);
    ICP_CUDA(cudaGetLastError());
    if (!with_ref && out->kl) ICP_CUDA(cudaMemsetAsync(out->kl, 0, sizeof(double) * N, st));
  }
  TokenArgs a;
  fill_token_args(a, shape, cfg, batch, adv);
  a.lp_cur_in = out->lp_cur;
  a.entropy_in = out->entropy;
  a.kl_in = with_ref ? out->kl : nullptr;
  a.kept = out->kept;
  a.calib = out->calib;
  a.surrogate = out->surrogate;
  a.coeff_d = out->coeff;
  a.block_stats = w.block_stats;
  const int grid = token_grid(N);
  k2_icepop_tokens<1><<<grid, TOK_THREADS, 0, st>>>(a);
  ICP_CUDA(cudaGetLastError());
  k_finalize_stats<<<1, 32 * ICEPOP_NSTATS, 0, st>>>(w.block_stats, grid, out->stats);
  k_merge_err<<<1, 1, 0, st>>>(w.err, out->stats);
  ICP_CUDA(cudaGetLastError());
  return ICEPOP_OK;
}

int icepop_bwd_f64(const icepop_shape* shape, const icepop_config* cfg, const double* hidden, const double* weight,
                   const double* weight_ref, const icepop_batch* batch, const icepop_f64_out* fwd, double grad_scale,
                   double* grad_hidden, double* grad_weight, int32_t accumulate, void* workspace,
                   size_t workspace_bytes, void* stream) {
  ICP_TRY(check_shape(shape, false));
  ICP_TRY(check_config(cfg));
  if (!fwd || !fwd->lse || !fwd->coeff) return fail(ICEPOP_EINVAL, "null forward outputs");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool kl_grad = weight_ref != nullptr && cfg->kl_coeff > 0.0;
  if (kl_grad && (!fwd->kl || !fwd->lse_ref || !batch))
    return fail(ICEPOP_EINVAL, "KL gradient needs kl, lse_ref and the batch geometry");
  F64Workspace w = carve_f64(shape, workspace, kl_grad);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(ICEPOP_EINVAL, "fp64 workspace too small: need %zu bytes", w.bytes);
  const int64_t N = shape->n_tokens, d = shape->hidden, V = shape->vocab;
  const bool dv = shape->weight_layout == ICEPOP_W_DV;
  if (N == 0) {
    if (grad_weight && !accumulate) ICP_CUDA(cudaMemsetAsync(grad_weight, 0, sizeof(double) * d * V, st));
    return ICEPOP_OK;
  }
  const int sg = std::min<int64_t>((N * V + 255) / 256, (int64_t)num_sms() * 16);
  ICP_TRY(logits_f64(shape, hidden, weight, w.Z, st));
  if (cfg->temperature != 1.0) k_scale_f64<<<sg, 256, 0, st>>>(w.Z, N * V, cfg->temperature);
  if (kl_grad) {
    ICP_TRY(logits_f64(shape, hidden, weight_ref, w.Zref, st));
    if (cfg->temperature != 1.0) k_scale_f64<<<sg, 256, 0, st>>>(w.Zref, N * V, cfg->temperature);
    k_kl_weight_f64<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(batch->cu_seqlens, shape->n_seqs,
                                                                 batch->group_offsets, shape->n_groups,
                                                                 shape->token_offset, N, cfg->kl_coeff,
                                                                 cfg->temperature, w.kw);
  }
  k_dz_f64<<<(unsigned)N, F64_ROW_THREADS, 0, st>>>(w.Z, kl_grad ? w.Zref : nullptr, V, batch ? batch->tokens : nullptr,
                                                    fwd->lse, kl_grad ? fwd->lse_ref : nullptr,
                                                    kl_grad ? fwd->kl : nullptr, fwd->coeff, kl_grad ? w.kw : nullptr,
                                                    grad_scale);
  ICP_CUDA(cudaGetLastError());
  if (grad_hidden) {
    // dH[t,f] = sum_v dZ[t,v] W(f,v)
    if (dv) ICP_TRY(gemm_f64(w.Z, V, 1, weight, 1, V, grad_hidden, d, N, d, V, 0, st));
    else ICP_TRY(gemm_f64(w.Z, V, 1, weight, d, 1, grad_hidden, d, N, d, V, 0, st));
  }
  if (grad_weight) {
    if (dv) ICP_TRY(gemm_f64(hidden, 1, d, w.Z, V, 1, grad_weight, V, d, V, N, accumulate, st));
    else ICP_TRY(gemm_f64(w.Z, 1, V, hidden, d, 1, grad_weight, d, V, d, N, accumulate, st));
  }
  return ICEPOP_OK;
}

int icepop_finish(const double* stats, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ICP_CUDA(cudaStreamSynchronize(st));
  double host_err = 0.0;
  ICP_CUDA(cudaMemcpy(&host_err, stats + ICEPOP_STAT_ERRORS, sizeof(double), cudaMemcpyDefault));
  const unsigned e = (unsigned)host_err;
  if (e & ERR_BAD_TOKEN) return fail(ICEPOP_EINVAL, "token id outside the vocabulary");
  if (e & ICEPOP_ERR_CALIB_OVERFLOW) return fail(ICEPOP_ENUMERIC, "calibration ratio overflow");
  if (e & ICEPOP_ERR_RATIO_OVERFLOW) return fail(ICEPOP_ENUMERIC, "importance ratio overflow");
  if (e & ICEPOP_ERR_NONFINITE) return fail(ICEPOP_ENUMERIC, "objective, gradient or update is not finite");
  return ICEPOP_OK;
}

int icepop_kl_bf16(const icepop_shape* shape, double temperature, const void* hidden, const void* weight_p,
                   const void* weight_q, float* kl, float* lse_p, float* lse_q, double* mean_kl, void* workspace,
                   size_t workspace_bytes, void* stream) {
  ICP_TRY(check_shape(shape, true));
  if (!(temperature > 0.0)) return fail(ICEPOP_EINVAL, "temperature must be positive");
  if (!hidden || !weight_p || !weight_q) return fail(ICEPOP_EINVAL, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  BF16Workspace w = carve_bf16(shape, workspace, 0, false, true);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(ICEPOP_EINVAL, "workspace too small: need %zu bytes", w.bytes);
  const int64_t N = shape->n_tokens, d = shape->hidden, V = shape->vocab;
  if (N == 0) return fail(ICEPOP_EINVAL, "probe set must be non-empty");  // discrepancy.py:136-137
  EpiParams ep;
  memset(&ep, 0, sizeof(ep));
  ep.scale_log2 = (float)(1.4426950408889634 / temperature);
  ep.inv_t = (float)(1.0 / temperature);
  ep.part = w.part;
  ep.ztok = w.ztok;
  const bool b_mn = shape->weight_layout == ICEPOP_W_DV;
  ICP_TRY(run_umma(EPI_LSE_REF, hidden, d, false, weight_p, b_mn ? V : d, b_mn, N, V, d, ep, st, Extent(), weight_q));
  const int grid = token_grid(N);
  k_kl_finish<<<grid, TOK_THREADS, 0, st>>>(w.part, (int)((V + bn_of(EPI_LSE_REF) - 1) / bn_of(EPI_LSE_REF)), N, kl,
                                            lse_p, lse_q, w.block_stats);
  if (mean_kl) k_sum_blocks<<<1, 32, 0, st>>>(w.block_stats, grid, 1.0 / (double)N, mean_kl);
  ICP_CUDA(cudaGetLastError());
  return ICEPOP_OK;
}

int icepop_sgd_update_f32(float* weight, const float* grad, float* velocity, void* weight_bf16, int64_t n, double lr,
                          double beta, double* stats, void* stream) {
  // objective.py:303-306, 320-321
  if (!(lr > 0.0)) return fail(ICEPOP_EINVAL, "learning rate must be positive");
  if (velocity && !(beta >= 0.0 && beta < 1.0)) return fail(ICEPOP_EINVAL, "momentum beta must be in [0, 1)");
  if (!weight || !grad || n < 0) return fail(ICEPOP_EINVAL, "null weight/grad");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0;
  ICP_CUDA(cudaGetDevice(&dev));
  int32_t* dg = nullptr;
  ICP_TRY(diag_ptr(dev, &dg));
  unsigned* e = reinterpret_cast<unsigned*>(dg + 2);  // the device pool's error word for this call
  ICP_CUDA(cudaMemsetAsync(e, 0, sizeof(unsigned), st));
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
  if (n > 0)
    k_sgd_update<<<std::max(grid, 1), 256, 0, st>>>(weight, grad, velocity,
                                                    static_cast<__nv_bfloat16*>(weight_bf16), n, (float)lr,
                                                    (float)beta, e);
  if (stats) {
    ICP_CUDA(cudaMemsetAsync(stats, 0, sizeof(double) * ICEPOP_NSTATS, st));
    k_merge_err<<<1, 1, 0, st>>>(e, stats);
  }
  ICP_CUDA(cudaGetLastError());
  return ICEPOP_OK;
}

int icepop_delta_gap_workspace_bytes(const icepop_shape* shape, int32_t f64, size_t* bytes) {
  ICP_TRY(check_shape(shape, !f64));
  if (!bytes) return fail(ICEPOP_EINVAL, "null out pointer");
  Carver c(nullptr);
  const size_t n = (size_t)std::max<int64_t>(shape->n_tokens, 1);
  c.take<uint8_t>(n * (size_t)shape->vocab * (f64 ? 8 : 4));  // train logits
  c.take<double>(2 * n);                                       // kl / gap rows when not requested
  *bytes = align_up(c.off, 256);
  return ICEPOP_OK;
}

// delta and max token gap (discrepancy.py:132-141) given the inference engine's logits: the train
// logits come from the lm_head GEMM (tcgen05 for bf16, SIMT for fp64), the rest from one fp64 row
// kernel and a fixed-order finish.
static int delta_gap_impl(const icepop_shape* shape, double temperature, const void* hidden, const void* weight,
                          const void* infer_logits, bool f64, double* kl_rows, double* gap_rows, double* delta,
                          double* max_gap, void* workspace, size_t workspace_bytes, void* stream) {
  ICP_TRY(check_shape(shape, !f64));
  if (!(temperature > 0.0)) return fail(ICEPOP_EINVAL, "temperature must be positive");
  const int64_t N = shape->n_tokens, d = shape->hidden, V = shape->vocab;
  if (N == 0) return fail(ICEPOP_EINVAL, "probe set must be non-empty");  // discrepancy.py:136-137
  if (!hidden || !weight || !infer_logits) return fail(ICEPOP_EINVAL, "null argument");
  size_t need = 0;
  ICP_TRY(icepop_delta_gap_workspace_bytes(shape, f64 ? 1 : 0, &need));
  if (!workspace || workspace_bytes < need) return fail(ICEPOP_EINVAL, "workspace too small: need %zu bytes", need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Carver c(workspace);
  void* z = c.take<uint8_t>((size_t)N * V * (f64 ? 8 : 4));
  double* rows = c.take<double>(2 * (size_t)N);
  double* kl = kl_rows ? kl_rows : rows;
  double* gap = gap_rows ? gap_rows : rows + N;
  const bool dv = shape->weight_layout == ICEPOP_W_DV;
  const int grid = (int)std::min<int64_t>(N, (int64_t)num_sms() * 8);
  if (f64) {
    ICP_TRY(logits_f64(shape, static_cast<const double*>(hidden), static_cast<const double*>(weight),
                       static_cast<double*>(z), st));
    k_delta_gap_rows<double, double><<<grid, DG_THREADS, 0, st>>>(
        static_cast<const double*>(z), static_cast<const double*>(infer_logits), N, V, 1.0 / temperature, kl, gap);
  } else {
    EpiParams ep;
    memset(&ep, 0, sizeof(ep));
    ep.out = z;
    ep.ldo = V;
    ep.out_f32 = 1;
    ep.vec_ok = (V % 8 == 0) ? 1 : 0;
    ICP_TRY(run_umma(EPI_STORE, hidden, d, false, weight, dv ? V : d, dv, N, V, d, ep, st));
    k_delta_gap_rows<float, float><<<grid, DG_THREADS, 0, st>>>(
        static_cast<const float*>(z), static_cast<const float*>(infer_logits), N, V, 1.0 / temperature, kl, gap);
  }
  ICP_CUDA(cudaGetLastError());
  k_delta_gap_finish<<<1, DG_THREADS, 0, st>>>(kl, gap, N, delta, max_gap);
  ICP_CUDA(cudaGetLastError());
  return ICEPOP_OK;
}

int icepop_delta_gap_bf16(const icepop_shape* shape, double temperature, const void* hidden, const void* weight,
                          const float* infer_logits, double* kl_rows, double* gap_rows, double* delta,
                          double* max_gap, void* workspace, size_t workspace_bytes, void* stream) {
  return delta_gap_impl(shape, temperature, hidden, weight, infer_logits, false, kl_rows, gap_rows, delta, max_gap,
                        workspace, workspace_bytes, stream);
}

int icepop_delta_gap_f64(const icepop_shape* shape, double temperature, const double* hidden, const double* weight,
                         const double* infer_logits, double* kl_rows, double* gap_rows, double* delta,
                         double* max_gap, void* workspace, size_t workspace_bytes, void* stream) {
  return delta_gap_impl(shape, temperature, hidden, weight, infer_logits, true, kl_rows, gap_rows, delta, max_gap,
                        workspace, workspace_bytes, stream);
}

int icepop_sgd_update_f64(double* weight_out, const double* weight, const double* grad, const double* velocity,
                          double* velocity_out, int64_t n, double lr, double beta, double* stats, void* stream) {
  // objective.py:301-326: lr <= 0 -> ValueError, beta outside [0, 1) -> ValueError
  if (!(lr > 0.0)) return fail(ICEPOP_EINVAL, "learning rate must be positive");
  if (velocity && !(beta >= 0.0 && beta < 1.0)) return fail(ICEPOP_EINVAL, "momentum beta must be in [0, 1)");
  if (!weight_out || !weight || !grad || n < 0 || (velocity && !velocity_out))
    return fail(ICEPOP_EINVAL, "null weight/grad/velocity_out");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0;
  ICP_CUDA(cudaGetDevice(&dev));
  int32_t* dg = nullptr;
  ICP_TRY(diag_ptr(dev, &dg));
  unsigned* e = reinterpret_cast<unsigned*>(dg + 3);
  ICP_CUDA(cudaMemsetAsync(e, 0, sizeof(unsigned), st));
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
  if (n > 0)
    k_sgd_update_f64<<<std::max(grid, 1), 256, 0, st>>>(weight_out, weight, grad, velocity, velocity_out, n, lr,
                                                         beta, e);
  if (stats) {
    ICP_CUDA(cudaMemsetAsync(stats, 0, sizeof(double) * ICEPOP_NSTATS, st));
    k_merge_err<<<1, 1, 0, st>>>(e, stats);
  }
  ICP_CUDA(cudaGetLastError());
  return ICEPOP_OK;
}

int icepop_wave_barrier_abandons(int64_t* count) {
  if (!count) return fail(ICEPOP_EINVAL, "null out pointer");
  int dev = 0;
  ICP_CUDA(cudaGetDevice(&dev));
  int32_t* d = nullptr;
  ICP_TRY(diag_ptr(dev, &d));
  int32_t h = 0;
  if (d) ICP_CUDA(cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost));
  *count = h;
  return ICEPOP_OK;
}

int icepop_set_cta_group(int32_t cta_group) {
  if (cta_group != 1 && cta_group != 2) return fail(ICEPOP_EINVAL, "cta_group must be 1 or 2");
  g_cta_group = cta_group;
  return ICEPOP_OK;
}

int icepop_set_wide_tiles(int32_t enable) {
  g_wide_tiles = enable <= 0 ? 0 : (enable >= 2 ? 2 : 1);
  return ICEPOP_OK;
}

int icepop_set_k1_wide(int32_t enable) {
  g_k1_wide = enable ? 1 : 0;
  return ICEPOP_OK;
}

int icepop_set_k1_run(int32_t run) {
  if (run < 0 || run > 64) return fail(ICEPOP_EINVAL, "k1 run length must be in [0, 64] (0 = automatic)");
  g_k1_run = run;
  return ICEPOP_OK;
}

int icepop_set_skip_inactive(int32_t enable) {
  g_skip_inactive = enable ? 1 : 0;
  return ICEPOP_OK;
}

int icepop_gemm_bf16(const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K, int32_t a_mn_major,
                     int32_t b_mn_major, int32_t c_f32, int32_t accumulate, void* stream) {
  if (!A || !B || !C) return fail(ICEPOP_EINVAL, "null operand");
  if (accumulate && !c_f32) return fail(ICEPOP_EINVAL, "accumulate needs an f32 output");
  EpiParams ep;
  memset(&ep, 0, sizeof(ep));
  ep.out = C;
  ep.ldo = N;
  ep.out_f32 = c_f32 ? 1 : 0;
  ep.accumulate = accumulate ? 1 : 0;
  ep.vec_ok = ((reinterpret_cast<uintptr_t>(C) & 15u) == 0) && (N % 8 == 0);
  // A: [M,K] (K-major) or [K,M]; B: [N,K] or [K,N]
  const int64_t lda = a_mn_major ? M : K;
  const int64_t ldb = b_mn_major ? N : K;
  return run_umma(EPI_STORE, A, lda, a_mn_major != 0, B, ldb, b_mn_major != 0, M, N, K, ep,
                  static_cast<cudaStream_t>(stream));
}

}  // extern "C"

// Load every kernel now (cudaFuncGetAttributes forces it under CUDA's lazy loading), not at its
// first launch: loading a function waits for the kernels running on the device, so a first
// launch behind a kernel that spins on another stream -- an NCCL kernel waiting on its peers --
// would wait for it and could deadlock.
template <int BN, bool A_MN, bool B_MN, int EPI, int CG>
static cudaError_t touch_gemm() {
  cudaFuncAttributes fa;
  return cudaFuncGetAttributes(&fa, umma_gemm_kernel<BN, A_MN, B_MN, EPI, CG>);
}

template <bool A_MN, bool B_MN, int EPI>
static int touch_epi() {  // the instantiations launch_umma can select
  constexpr int BN = epi_dual(EPI) ? 128 : BN_;
  cudaError_t e = touch_gemm<BN, A_MN, B_MN, EPI, 2>();
  if (e == cudaSuccess) e = touch_gemm<BN, A_MN, B_MN, EPI, 1>();
  if constexpr (EPI == EPI_STORE || EPI == EPI_LSE)
    if (e == cudaSuccess) e = touch_gemm<BN_WIDE, A_MN, B_MN, EPI, 2>();
  if (e != cudaSuccess) return fail(ICEPOP_ECUDA, "kernel load failed: %s", cudaGetErrorString(e));
  return ICEPOP_OK;
}

template <class K>
static int touch(K k) {
  cudaFuncAttributes fa;
  const cudaError_t e = cudaFuncGetAttributes(&fa, k);
  if (e != cudaSuccess) return fail(ICEPOP_ECUDA, "kernel load failed: %s", cudaGetErrorString(e));
  return ICEPOP_OK;
}

static int preload_kernels() {
  ICP_TRY((touch_epi<false, false, EPI_STORE>()));
  ICP_TRY((touch_epi<false, true, EPI_STORE>()));
  ICP_TRY((touch_epi<true, false, EPI_STORE>()));
  ICP_TRY((touch_epi<true, true, EPI_STORE>()));
  ICP_TRY((touch_epi<false, false, EPI_LSE>()));
  ICP_TRY((touch_epi<false, true, EPI_LSE>()));
  ICP_TRY((touch_epi<false, false, EPI_DZ>()));
  ICP_TRY((touch_epi<false, true, EPI_DZ>()));
  ICP_TRY((touch_epi<false, false, EPI_LSE_REF>()));
  ICP_TRY((touch_epi<false, true, EPI_LSE_REF>()));
  ICP_TRY((touch_epi<false, false, EPI_DZ_REF>()));
  ICP_TRY((touch_epi<false, true, EPI_DZ_REF>()));
  ICP_TRY(touch(k0_group_advantages));
  ICP_TRY(touch(k2_icepop_tokens<0>));
  ICP_TRY(touch(k2_icepop_tokens<1>));
  ICP_TRY(touch(k2_icepop_tokens<2>));
  ICP_TRY(touch(k2_icepop_tokens<3>));
  ICP_TRY(touch(k_finalize_stats));
  ICP_TRY(touch(k_merge_err));
  ICP_TRY(touch(k_check_tokens));
  ICP_TRY(touch(k_logprob_finish));
  ICP_TRY(touch(k_kl_finish));
  ICP_TRY(touch(k_sum_blocks));
  ICP_TRY(touch(k_sgd_update));
  ICP_TRY(touch(k_sgd_update_f64));
  ICP_TRY(touch(k_delta_gap_rows<float, float>));
  ICP_TRY(touch(k_delta_gap_rows<double, double>));
  ICP_TRY(touch(k_delta_gap_finish));
  ICP_TRY(touch(k_rs_fold));
  ICP_TRY(touch(k_active_count));
  ICP_TRY(touch(k_active_scan));
  ICP_TRY(touch(k_active_scatter));
  ICP_TRY(touch(k_gather_active));
  ICP_TRY(touch(k_dz_probs));
  ICP_TRY(touch(k_block_flags));
  ICP_TRY(touch(k_block_lists));
  ICP_TRY(touch(k_sp_prep));
  ICP_TRY(touch(k_transpose_rows));
  ICP_TRY(touch(k_iota));
  ICP_TRY(touch(k_onehot_scatter));
  // CUB's radix sort (the one-hot scatter's order): run a small and a large sort once so that
  // both of its dispatch paths (single tile, one-sweep) are loaded
  const int n_big = 1 << 20;
  int32_t* buf = nullptr;
  size_t tb_small = 0, tb_big = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb_small, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, 64, 0, 18);
  cub::DeviceRadixSort::SortPairs(nullptr, tb_big, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, n_big, 0, 18);
  const size_t tb = std::max(tb_small, tb_big);
  ICP_CUDA(cudaMalloc(&buf, 4 * (size_t)n_big * sizeof(int32_t) + tb));
  ICP_CUDA(cudaMemset(buf, 0, 4 * (size_t)n_big * sizeof(int32_t)));
  void* tmp = buf + 4 * (size_t)n_big;
  for (int n : {64, n_big}) {
    size_t t = tb;
    ICP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t, buf, buf + n_big, buf + 2 * n_big, buf + 3 * n_big, n, 0, 18,
                                             (cudaStream_t)0));
  }
  ICP_CUDA(cudaDeviceSynchronize());
  ICP_CUDA(cudaFree(buf));
  return ICEPOP_OK;
}
