/*
 * One IcePop fwd+bwd step through the C ABI alone (include/icepop.h): no Python, no torch.
 * This is what a non-Python caller of the reference's hot path (objective.py:172-298) links.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_api_example.c \
 *       -L paper_2510_18855_b200 -licepop_b200 -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2510_18855_b200 -o build/c_api_example
 *   build/c_api_example [dump.bin]
 *
 * Inputs are a seeded synthetic batch (4 rollouts in 2 prompt groups, bf16 hidden/weight in
 * the lm_head [V, d] layout, rewards -> K0 advantages). The forward keeps the bf16
 * probabilities (stored-probabilities mode) and the backward forms dZ from them in place.
 * Prints the statistics and a checksum; with a path argument it also dumps inputs and
 * outputs (tests/test_c_api.py replays them through the Python layer and compares bits).
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "icepop.h"

#define N_SEQS 4
#define SEQ_LEN 250
#define N_TOK (N_SEQS * SEQ_LEN)
#define HID 256
#define VOCAB 2048

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));         \
      return 1;                                                                          \
    }                                                                                    \
  } while (0)
#define IK(x)                                                                            \
  do {                                                                                   \
    int r_ = (x);                                                                        \
    if (r_ != ICEPOP_OK) {                                                               \
      fprintf(stderr, "%s:%d icepop error %d: %s\n", __FILE__, __LINE__, r_, icepop_last_error()); \
      return 2;                                                                          \
    }                                                                                    \
  } while (0)

static uint64_t g_state = 0x9E3779B97F4A7C15ull;
static double uniform(void) { /* splitmix64 -> [0, 1) */
  uint64_t z = (g_state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}
static double normal(void) { /* Box-Muller */
  double u1 = uniform(), u2 = uniform();
  if (u1 < 1e-300) u1 = 1e-300;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}
static uint16_t to_bf16(float f) { /* round to nearest even */
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

int main(int argc, char** argv) {
  IK(icepop_device_check(0));
  const size_t nh = (size_t)N_TOK * HID, nw = (size_t)VOCAB * HID;
  uint16_t* h_hid = malloc(nh * 2);
  uint16_t* h_w = malloc(nw * 2);
  int32_t tokens[N_TOK], cu[N_SEQS + 1], go[3] = {0, 2, 4};
  double lp_old[N_TOK], lp_inf[N_TOK], rewards[N_SEQS] = {1.0, 0.0, 0.0, 1.0};
  for (size_t i = 0; i < nh; ++i) h_hid[i] = to_bf16((float)normal());
  for (size_t i = 0; i < nw; ++i) h_w[i] = to_bf16((float)(normal() * 2.0 / sqrt((double)HID)));
  for (int t = 0; t < N_TOK; ++t) {
    tokens[t] = (int32_t)(uniform() * VOCAB);
    lp_old[t] = -log((double)VOCAB) + 0.5 * normal();
    lp_inf[t] = lp_old[t] - 0.3 * normal();
  }
  for (int s = 0; s <= N_SEQS; ++s) cu[s] = s * SEQ_LEN;

  /* device buffers */
  void *d_hid, *d_w, *d_probs, *d_gh, *d_fws, *d_bws;
  int32_t *d_tok, *d_cu, *d_go;
  double *d_lpo, *d_lpi, *d_rew, *d_lp, *d_calib, *d_sur, *d_stats;
  float *d_lse, *d_ent, *d_coeff, *d_tmax, *d_gw;
  uint8_t* d_kept;
  CK(cudaMalloc(&d_hid, nh * 2));
  CK(cudaMalloc(&d_w, nw * 2));
  CK(cudaMalloc((void**)&d_tok, sizeof tokens));
  CK(cudaMalloc((void**)&d_cu, sizeof cu));
  CK(cudaMalloc((void**)&d_go, sizeof go));
  CK(cudaMalloc((void**)&d_lpo, sizeof lp_old));
  CK(cudaMalloc((void**)&d_lpi, sizeof lp_inf));
  CK(cudaMalloc((void**)&d_rew, sizeof rewards));
  CK(cudaMalloc((void**)&d_lse, N_TOK * 4));
  CK(cudaMalloc((void**)&d_ent, N_TOK * 4));
  CK(cudaMalloc((void**)&d_coeff, N_TOK * 4));
  CK(cudaMalloc((void**)&d_lp, N_TOK * 8));
  CK(cudaMalloc((void**)&d_calib, N_TOK * 8));
  CK(cudaMalloc((void**)&d_sur, N_TOK * 8));
  CK(cudaMalloc((void**)&d_kept, N_TOK));
  CK(cudaMalloc((void**)&d_stats, ICEPOP_NSTATS * 8));
  CK(cudaMalloc(&d_probs, (size_t)N_TOK * VOCAB * 2));
  CK(cudaMalloc((void**)&d_tmax, (size_t)N_TOK * ICEPOP_TILE_MAX_LD(VOCAB) * 4));
  CK(cudaMalloc(&d_gh, nh * 2));
  CK(cudaMalloc((void**)&d_gw, nw * 4));
  CK(cudaMemcpy(d_hid, h_hid, nh * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_w, h_w, nw * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_tok, tokens, sizeof tokens, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_cu, cu, sizeof cu, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_go, go, sizeof go, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_lpo, lp_old, sizeof lp_old, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_lpi, lp_inf, sizeof lp_inf, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_rew, rewards, sizeof rewards, cudaMemcpyHostToDevice));

  icepop_shape shape = {N_TOK, 0, HID, VOCAB, N_SEQS, 2, ICEPOP_W_VD, 0};
  icepop_config cfg = {0.5, 5.0, 0.2, 2.0, 1.0, 0.0, ICEPOP_ALGO_ICEPOP, 0};
  icepop_batch batch = {d_tok, d_lpo, d_lpi, d_cu, d_go, NULL, d_rew};
  size_t fwd_bytes = 0, bwd_bytes = 0;
  IK(icepop_workspace_bytes(&shape, 0, 0, &fwd_bytes, NULL));
  IK(icepop_workspace_bytes(&shape, -1, 0, NULL, &bwd_bytes)); /* stored-probabilities backward */
  CK(cudaMalloc(&d_fws, fwd_bytes));
  CK(cudaMalloc(&d_bws, bwd_bytes));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));

  icepop_fwd_out out;
  memset(&out, 0, sizeof out);
  out.lse = d_lse;
  out.lp_cur = d_lp;
  out.entropy = d_ent;
  out.kept = d_kept;
  out.calib = d_calib;
  out.surrogate = d_sur;
  out.coeff = d_coeff;
  out.stats = d_stats;
  out.probs = d_probs;
  out.tile_max = d_tmax;
  IK(icepop_fwd_bf16(&shape, &cfg, d_hid, d_w, NULL, &batch, &out, d_fws, fwd_bytes, st));

  icepop_saved saved;
  memset(&saved, 0, sizeof saved);
  saved.tokens = d_tok;
  saved.lse = d_lse;
  saved.coeff = d_coeff;
  saved.probs = d_probs;
  saved.tile_max = d_tmax;
  saved.lp_cur = d_lp; /* the sampled token's exact term c (1 - exp(lp_cur)) */
  /* loss = -J: grad_scale = -1; the workspace lets the backward compact zero-coefficient rows */
  IK(icepop_bwd_bf16(&shape, &cfg, d_hid, d_w, NULL, &saved, -1.0, d_gh, 0, d_gw, 0, d_bws, bwd_bytes, st));
  IK(icepop_finish(d_stats, st));

  double stats[ICEPOP_NSTATS];
  float* gw = malloc(nw * 4);
  CK(cudaMemcpy(stats, d_stats, sizeof stats, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(gw, d_gw, nw * 4, cudaMemcpyDeviceToHost));
  double l1 = 0.0;
  for (size_t i = 0; i < nw; ++i) l1 += fabs((double)gw[i]);
  printf("objective=%.17g popped=%.0f tokens=%.0f grad_weight_l1=%.17g\n", stats[ICEPOP_STAT_OBJECTIVE],
         stats[ICEPOP_STAT_N_POPPED], stats[ICEPOP_STAT_TOKENS], l1);

  if (argc > 1) { /* inputs then outputs, raw little-endian */
    FILE* f = fopen(argv[1], "wb");
    if (!f) return 3;
    fwrite(h_hid, 2, nh, f);
    fwrite(h_w, 2, nw, f);
    fwrite(tokens, 4, N_TOK, f);
    fwrite(lp_old, 8, N_TOK, f);
    fwrite(lp_inf, 8, N_TOK, f);
    fwrite(stats, 8, ICEPOP_NSTATS, f);
    fwrite(gw, 4, nw, f);
    fclose(f);
  }
  free(h_hid);
  free(h_w);
  free(gw);
  return 0;
}
