/*
 * CPU oracle — TEST INFRASTRUCTURE ONLY (see oracle.h for scope and parity status).
 * Build: gcc -O3 -fopenmp -ffp-contract=off (no FMA contraction: the fp64 GEMM must add in
 * exactly the order of infersim::exec_reference, gemm.hpp:147-202).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ fp16 */
uint16_t or_f32_to_f16(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const uint32_t absx = x & 0x7fffffffu;
  if (absx >= 0x7f800000u) return (uint16_t)(sign | (absx > 0x7f800000u ? 0x7e00u : 0x7c00u));
  if (absx >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u);
  if (absx < 0x38800000u) {
    if (absx < 0x33000000u) return (uint16_t)sign;
    const uint32_t e = absx >> 23;
    const uint32_t m = (absx & 0x7fffffu) | 0x800000u;
    const uint32_t shift = 126 - e;
    uint32_t q = m >> shift;
    const uint32_t rem = m & ((1u << shift) - 1u);
    const uint32_t half = 1u << (shift - 1);
    if (rem > half || (rem == half && (q & 1u))) ++q;
    return (uint16_t)(sign | q);
  }
  uint32_t h = (((absx >> 23) - 112) << 10) | ((absx >> 13) & 0x3ffu);
  const uint32_t rem = absx & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
  return (uint16_t)(sign | h);
}

float or_f16_to_f32(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1fu, m = h & 0x3ffu;
  uint32_t out;
  if (e == 0) {
    if (m == 0) {
      out = sign;
    } else {
      float f = (float)m * (1.0f / 16777216.0f);
      memcpy(&out, &f, 4);
      out |= sign;
    }
  } else if (e == 31) {
    out = sign | 0x7f800000u | (m << 13);
  } else {
    out = sign | ((e + 112) << 23) | (m << 13);
  }
  float r;
  memcpy(&r, &out, 4);
  return r;
}

static float f16r(float v) { return or_f16_to_f32(or_f32_to_f16(v)); }
double or_round_f16(double v) { return (double)f16r((float)v); }

/* ------------------------------------------------------------------ synthetic weights */
static uint64_t sm64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t or_synth_base(uint64_t seed, int32_t layer, int32_t tensor) {
  return sm64(seed ^ (0x51ED2701ull * (uint64_t)(layer + 1)) ^ ((uint64_t)tensor << 56));
}
float or_synth_unit(uint64_t base, uint64_t flat) {
  const uint64_t h = sm64(base + flat);
  const int32_t u24 = (int32_t)(h >> 40);
  return (float)(2 * u24 - (1 << 24)) * (1.0f / 16777216.0f);
}

/* tensor ids and amplitudes: include/dsinf.h DSINF_T_*, csrc/synth.h SynthScale */
enum { T_QKV = 1, T_QKV_B, T_O, T_O_B, T_UP, T_UP_B, T_DOWN, T_DOWN_B, T_LN1_G, T_LN1_B, T_LN2_G, T_LN2_B, T_WTE, T_LNF_G, T_LNF_B };
static const float kAmpW = 0.034641016f, kAmpB = 0.017320508f, kAmpG = 0.1f, kAmpBeta = 0.05f;

static float synth_w(uint64_t base, uint64_t flat, float amp) {
  const float u = or_synth_unit(base, flat);
  const float w = u * amp;
  return f16r(w);
}
static float synth_v(uint64_t base, uint64_t flat, float offset, float amp) {
  const float u = or_synth_unit(base, flat);
  const float t = u * amp;
  return f16r(offset + t);
}

/* ------------------------------------------------------------------ gemm.hpp restatement */
int32_t or_cache_line_pack(int32_t dtype_bytes) { /* gemm.hpp:57-60 */
  int32_t m = 128 / (32 * dtype_bytes);
  return m < 1 ? 1 : (m > 4 ? 4 : m);
}

int or_derive_schedule(int64_t N, int64_t K, int64_t B, int32_t dtype_bytes, int32_t sm_count, or_schedule* s) {
  /* gemm.hpp:65-96 */
  if (N < 1 || K < 1 || B < 1) return 2;
  if (dtype_bytes != 1 && dtype_bytes != 2 && dtype_bytes != 4) return 2;
  s->pack_M = or_cache_line_pack(dtype_bytes);
  s->output_tiles = (N + 31) / 32;
  const int64_t groups = (K + s->pack_M - 1) / s->pack_M;
  int64_t w = groups / 32;
  s->warps_per_block = (int32_t)(w < 1 ? 1 : (w > 8 ? 8 : w));
  s->two_d = 0;
  s->input_tiles = 1;
  s->kernel_count = 1;
  if (s->output_tiles >= sm_count) return 0;
  int64_t tiles = 1;
  while (s->output_tiles * tiles < sm_count && tiles * 2 <= groups) tiles *= 2;
  if (tiles == 1) return 0;
  s->two_d = 1;
  s->input_tiles = tiles;
  s->kernel_count = 2;
  return 0;
}

int64_t or_packed_index(int64_t n, int64_t k, int64_t N, int32_t M) { /* gemm.hpp:108-111 */
  return (k / M) * (N * M) + n * M + (k % M);
}

void or_pack(const double* W, int64_t N, int64_t K, int32_t M, double* out) { /* gemm.hpp:113-130 */
  const int64_t kp = (K + M - 1) / M * M;
  memset(out, 0, sizeof(double) * (size_t)(N * kp));
  for (int64_t n = 0; n < N; ++n)
    for (int64_t k = 0; k < K; ++k) out[or_packed_index(n, k, N, M)] = W[n * K + k];
}

int or_exec_sameorder(const double* packed, int64_t N, int64_t K, int32_t M, const or_schedule* s,
                      const double* x, int64_t B, double* out) {
  /* gemm.hpp:147-202: per output, warps accumulate contiguous K slices sequentially, warp
   * partials are summed in warp order, then input-tile partials in tile order. */
  if (B < 1) return 2;
  const int64_t kp = (K + M - 1) / M * M;
  const int64_t tiles = s->two_d ? s->input_tiles : 1;
  const int64_t tile_k = (kp + tiles - 1) / tiles;
  const int warps = s->warps_per_block < 1 ? 1 : s->warps_per_block;
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < N; ++n) {
    for (int64_t b = 0; b < B; ++b) {
      double result = 0.0;
      for (int64_t it = 0; it < tiles; ++it) {
        const int64_t kb = it * tile_k;
        const int64_t ke = (kb + tile_k < kp) ? kb + tile_k : kp;
        const int64_t span = ke - kb;
        const int64_t per = (span + warps - 1) / warps;
        double tile_sum = 0.0;
        for (int w = 0; w < warps; ++w) {
          const int64_t wb = kb + w * per;
          const int64_t we = (wb + per < ke) ? wb + per : ke;
          double acc = 0.0;
          for (int64_t kk = wb; kk < we; ++kk) {
            const double wv = packed[or_packed_index(n, kk, N, M)];
            const double xv = kk < K ? x[b * K + kk] : 0.0;
            acc += wv * xv;
          }
          tile_sum += acc;
        }
        result += tile_sum;
      }
      out[b * N + n] = result;
    }
  }
  return 0;
}

void or_gemm_f64(const float* W, int64_t N, int64_t K, const or_schedule* s, const double* x, int64_t B,
                 double* out) {
  const int32_t M = s->pack_M;
  const int64_t kp = (K + M - 1) / M * M;
  const int64_t tiles = s->two_d ? s->input_tiles : 1;
  const int64_t tile_k = (kp + tiles - 1) / tiles;
  const int warps = s->warps_per_block < 1 ? 1 : s->warps_per_block;
  double* xt = (double*)malloc(sizeof(double) * (size_t)(kp * B)); /* [kp][B], zero pad */
  for (int64_t k = 0; k < kp; ++k)
    for (int64_t b = 0; b < B; ++b) xt[k * B + b] = k < K ? x[b * K + k] : 0.0;
#pragma omp parallel
  {
    double* acc = (double*)malloc(sizeof(double) * (size_t)B * 3);
    double* tsum = acc + B;
    double* res = acc + 2 * B;
#pragma omp for schedule(static)
    for (int64_t n = 0; n < N; ++n) {
      const float* row = W + n * K;
      for (int64_t b = 0; b < B; ++b) res[b] = 0.0;
      for (int64_t it = 0; it < tiles; ++it) {
        const int64_t kb = it * tile_k;
        const int64_t ke = (kb + tile_k < kp) ? kb + tile_k : kp;
        const int64_t per = (ke - kb + warps - 1) / warps;
        for (int64_t b = 0; b < B; ++b) tsum[b] = 0.0;
        for (int w = 0; w < warps; ++w) {
          const int64_t wb = kb + w * per;
          const int64_t we = (wb + per < ke) ? wb + per : ke;
          for (int64_t b = 0; b < B; ++b) acc[b] = 0.0;
          for (int64_t kk = wb; kk < we; ++kk) {
            const double wv = kk < K ? (double)row[kk] : 0.0;
            const double* xk = xt + kk * B;
            for (int64_t b = 0; b < B; ++b) acc[b] += wv * xk[b];
          }
          for (int64_t b = 0; b < B; ++b) tsum[b] += acc[b];
        }
        for (int64_t b = 0; b < B; ++b) res[b] += tsum[b];
      }
      for (int64_t b = 0; b < B; ++b) out[b * N + n] = res[b];
    }
    free(acc);
  }
  free(xt);
}

/* ------------------------------------------------------------------ INT8 */
static float q_scale(float maxabs) { return maxabs > 0.0f ? maxabs / 127.0f : 1.0f; }
static int8_t q_one(float x, float s) {
  const float r = x / s;
  float q = nearbyintf(r); /* round half to even (default rounding mode) */
  if (q > 127.0f) q = 127.0f;
  if (q < -127.0f) q = -127.0f;
  return (int8_t)q;
}

void or_quant_rows(const float* x, int64_t rows, int64_t K, int8_t* q, float* scales) {
#pragma omp parallel for schedule(static) if (rows * K > (1 << 20))
  for (int64_t r = 0; r < rows; ++r) {
    float mx = 0.0f;
    for (int64_t k = 0; k < K; ++k) {
      const float a = fabsf(x[r * K + k]);
      if (a > mx) mx = a;
    }
    const float s = q_scale(mx);
    scales[r] = s;
    for (int64_t k = 0; k < K; ++k) q[r * K + k] = q_one(x[r * K + k], s);
  }
}

/* K-group quantisation (dsinf_quantize_weights_int8_groups; SURVEY §8c K-group recipe, group = 128):
 * per (row, group) s = fp16(max|w| / 127) (fp32 divide, round to nearest even; 1 for an all-zero or
 * fp16-underflowing group), q = clamp(rint(w / s), +-127) with an fp32 divide by the fp16 scale.
 * scales_f16 [ceil(K/group)][rows] as fp16 bits. */
void or_quant_groups(const float* x, int64_t rows, int64_t K, int64_t group, int8_t* q, uint16_t* scales_f16) {
  const int64_t G = (K + group - 1) / group;
#pragma omp parallel for schedule(static) if (rows * K > (1 << 20))
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t g = 0; g < G; ++g) {
      const int64_t k0 = g * group, k1 = k0 + group < K ? k0 + group : K;
      float mx = 0.0f;
      for (int64_t k = k0; k < k1; ++k) {
        const float a = fabsf(x[r * K + k]);
        if (a > mx) mx = a;
      }
      uint16_t sh = or_f32_to_f16(q_scale(mx));
      if (or_f16_to_f32(sh) == 0.0f) sh = or_f32_to_f16(1.0f);
      scales_f16[g * rows + r] = sh;
      const float s = or_f16_to_f32(sh);
      for (int64_t k = k0; k < k1; ++k) q[r * K + k] = q_one(x[r * K + k], s);
    }
}

void or_gemm_i8(const int8_t* wq, const float* ws, const int8_t* xq, const float* xs, int64_t N, int64_t K,
                int64_t B, int32_t* acc, float* y) {
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < N; ++n) {
    const int8_t* row = wq + n * K;
    for (int64_t b = 0; b < B; ++b) {
      const int8_t* xr = xq + b * K;
      int64_t a = 0;
      for (int64_t k = 0; k < K; ++k) a += (int32_t)row[k] * (int32_t)xr[k];
      const int32_t a32 = (int32_t)a;
      if (acc) acc[b * N + n] = a32;
      if (y) {
        const float t = (float)a32 * xs[b];
        y[b * N + n] = t * ws[n];
      }
    }
  }
}

/* ------------------------------------------------------------------ decoder model */
typedef struct {
  float *wqkv, *wo, *wup, *wdown, *wlm;       /* fp16 path: row-major local shards */
  int8_t *qqkv, *qo, *qup, *qdown;             /* int8 path */
  float *gqkv, *go, *gup, *gdown;              /* int8 K-group scales [Kl/128][Nl] (fp16 values), or NULL */
  float *sqkv, *so, *sup, *sdown;              /* int8 row scales (global-row) */
} or_rank_w;

typedef struct {
  or_rank_w* ranks; /* [tp] */
  float *bqkv, *bo, *bup, *bdown;               /* global vectors */
  float *ln1g, *ln1b, *ln2g, *ln2b;
} or_layer;

struct or_model {
  or_config c;
  int64_t h, L, H, d, Hl, V, Vpad, Vl, F, Fl;
  int t, B;
  or_layer* layers;
  float *wte, *lnfg, *lnfb;   /* wte [V][h]; LM rank shards in layers? kept per rank below */
  float** wlm;                /* [t] -> [Vl][h] */
  float* rope;                /* [max_ctx][d/2][2] */
  float *kc, *vc;             /* [L][B][H][max_ctx][d] */
  float* res;                 /* [B][h] */
  float* final_hidden;        /* [B][h] */
  or_gemm_hook_fn hook;       /* optional fp16-path GEMM (the reference's exec_reference) */
  void* hook_ctx;
};

void or_model_set_int8_act(or_model* m, int32_t int8_act) { m->c.int8_act = int8_act; }

void or_model_set_gemm_hook(or_model* m, or_gemm_hook_fn fn, void* ctx) {
  m->hook = fn;
  m->hook_ctx = ctx;
}

static float* falloc(int64_t n) { return (float*)calloc((size_t)(n > 0 ? n : 1), sizeof(float)); }

/* global [rows][cols] tensor value */
static float gval(uint64_t base, int64_t row, int64_t col, int64_t cols) { return synth_w(base, (uint64_t)(row * cols + col), kAmpW); }

static void gen_vec(float* out, int64_t n, uint64_t base, float offset, float amp) {
  for (int64_t i = 0; i < n; ++i) out[i] = synth_v(base, (uint64_t)i, offset, amp);
}

/* Fill a local [Nl][Kl] shard of a global [Ng][Kg] matrix: local row n -> global row via
 * (n / sec_l) * sec_g + row_off + n % sec_l, local col k -> col_off + k. */
static void gen_shard(float* out, int64_t Nl, int64_t Kl, int64_t Kg, int64_t sec_l, int64_t sec_g, int64_t row_off,
                      int64_t col_off, int64_t valid_rows, uint64_t base) {
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < Nl; ++n) {
    const int64_t gr = (n / sec_l) * sec_g + row_off + n % sec_l;
    for (int64_t k = 0; k < Kl; ++k) out[n * Kl + k] = gr < valid_rows ? gval(base, gr, col_off + k, Kg) : 0.0f;
  }
}

/* int8 shard with scales over the FULL global row */
static void gen_shard_i8(int8_t* q, float* scales, int64_t Nl, int64_t Kl, int64_t Kg, int64_t sec_l, int64_t sec_g,
                         int64_t row_off, int64_t col_off, uint64_t base) {
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < Nl; ++n) {
    const int64_t gr = (n / sec_l) * sec_g + row_off + n % sec_l;
    float mx = 0.0f;
    for (int64_t k = 0; k < Kg; ++k) {
      const float a = fabsf(gval(base, gr, k, Kg));
      if (a > mx) mx = a;
    }
    const float s = q_scale(mx);
    scales[n] = s;
    for (int64_t k = 0; k < Kl; ++k) q[n * Kl + k] = q_one(gval(base, gr, col_off + k, Kg), s);
  }
}

/* K-group variant (or_config.int8_group = 128; ops.cu init_packed_i8_groups_kernel): per (global row,
 * 128-k group of the global k index) s = fp16(max|w| / 127), q = clamp(rint(w / s)); the local
 * k range starts at col_off (a multiple of 128).  gs [Kl/128][Nl] holds the fp16 scales as floats. */
static void gen_shard_i8_groups(int8_t* q, float* gs, int64_t Nl, int64_t Kl, int64_t Kg, int64_t sec_l,
                                int64_t sec_g, int64_t row_off, int64_t col_off, uint64_t base) {
  const int64_t G = Kl / 128;
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < Nl; ++n) {
    const int64_t gr = (n / sec_l) * sec_g + row_off + n % sec_l;
    for (int64_t g = 0; g < G; ++g) {
      float mx = 0.0f;
      for (int64_t k = g * 128; k < g * 128 + 128; ++k) {
        const float a = fabsf(gval(base, gr, col_off + k, Kg));
        if (a > mx) mx = a;
      }
      uint16_t sh = or_f32_to_f16(q_scale(mx));
      if (or_f16_to_f32(sh) == 0.0f) sh = or_f32_to_f16(1.0f);
      const float sc = or_f16_to_f32(sh);
      gs[g * Nl + n] = sc;
      for (int64_t k = g * 128; k < g * 128 + 128; ++k) q[n * Kl + k] = q_one(gval(base, gr, col_off + k, Kg), sc);
    }
  }
}

/* Whole global tensors for the sequence oracle (oracle/seq_oracle.py): the same values the
 * per-rank shards above take (gval / synth_v), rows >= valid_rows zero. */
void or_synth_matrix(uint64_t seed, int32_t layer, int32_t tensor, int64_t rows, int64_t cols, int64_t valid_rows,
                     float* out) {
  gen_shard(out, rows, cols, cols, rows, rows, 0, 0, valid_rows, or_synth_base(seed, layer, tensor));
}

void or_synth_vector(uint64_t seed, int32_t layer, int32_t tensor, int64_t n, float* out) {
  float offset = 0.f, amp = kAmpB;
  if (tensor == T_LN1_G || tensor == T_LN2_G || tensor == T_LNF_G) {
    offset = 1.f;
    amp = kAmpG;
  } else if (tensor == T_LN1_B || tensor == T_LN2_B || tensor == T_LNF_B) {
    amp = kAmpBeta;
  }
  gen_vec(out, n, or_synth_base(seed, layer, tensor), offset, amp);
}

or_model* or_model_create(const or_config* cfg) {
  or_model* m = (or_model*)calloc(1, sizeof(or_model));
  m->c = *cfg;
  if (m->c.ln_eps <= 0.f) m->c.ln_eps = 1e-5f;
  if (m->c.rope_base <= 0.f) m->c.rope_base = 10000.f;
  if (m->c.sm_count <= 0) m->c.sm_count = 148;
  m->h = cfg->hidden;
  m->L = cfg->layers;
  m->H = cfg->heads;
  m->d = m->h / m->H;
  m->t = cfg->tp < 1 ? 1 : cfg->tp;
  m->Hl = m->H / m->t;
  m->V = cfg->vocab;
  const int64_t vq = 128LL * m->t;
  m->Vpad = (m->V + vq - 1) / vq * vq;
  m->Vl = m->Vpad / m->t;
  m->F = 4 * m->h;
  m->Fl = m->F / m->t;
  m->B = cfg->batch;
  const int64_t h = m->h, Hl = m->Hl, d = m->d, Fl = m->Fl;
  const int i8 = cfg->dtype_bytes == 1;
  const uint64_t seed = cfg->seed;
  m->layers = (or_layer*)calloc((size_t)(m->L > 0 ? m->L : 1), sizeof(or_layer));
  for (int64_t l = 0; l < m->L; ++l) {
    or_layer* ly = &m->layers[l];
    const int li = (int)l;
    ly->ranks = (or_rank_w*)calloc((size_t)m->t, sizeof(or_rank_w));
    for (int r = 0; r < m->t; ++r) {
      or_rank_w* w = &ly->ranks[r];
      const uint64_t bq = or_synth_base(seed, li, T_QKV), bo = or_synth_base(seed, li, T_O);
      const uint64_t bu = or_synth_base(seed, li, T_UP), bd = or_synth_base(seed, li, T_DOWN);
      if (!i8) {
        w->wqkv = falloc(3 * Hl * d * h);
        gen_shard(w->wqkv, 3 * Hl * d, h, h, Hl * d, h, r * Hl * d, 0, 3 * h, bq);
        w->wo = falloc(h * Hl * d);
        gen_shard(w->wo, h, Hl * d, h, h, h, 0, r * Hl * d, h, bo);
        w->wup = falloc(Fl * h);
        gen_shard(w->wup, Fl, h, h, Fl, m->F, r * Fl, 0, m->F, bu);
        w->wdown = falloc(h * Fl);
        gen_shard(w->wdown, h, Fl, m->F, h, h, 0, r * Fl, h, bd);
      } else {
        w->qqkv = (int8_t*)malloc((size_t)(3 * Hl * d * h));
        w->sqkv = falloc(3 * Hl * d);
        gen_shard_i8(w->qqkv, w->sqkv, 3 * Hl * d, h, h, Hl * d, h, r * Hl * d, 0, bq);
        w->qo = (int8_t*)malloc((size_t)(h * Hl * d));
        w->so = falloc(h);
        gen_shard_i8(w->qo, w->so, h, Hl * d, h, h, h, 0, r * Hl * d, bo);
        w->qup = (int8_t*)malloc((size_t)(Fl * h));
        w->sup = falloc(Fl);
        gen_shard_i8(w->qup, w->sup, Fl, h, h, Fl, m->F, r * Fl, 0, bu);
        w->qdown = (int8_t*)malloc((size_t)(h * Fl));
        w->sdown = falloc(h);
        gen_shard_i8(w->qdown, w->sdown, h, Fl, m->F, h, h, 0, r * Fl, bd);
        if (m->c.int8_group == 128) {  /* K-group weights replace the row-scaled ones */
          w->gqkv = falloc(3 * Hl * d * (h / 128));
          gen_shard_i8_groups(w->qqkv, w->gqkv, 3 * Hl * d, h, h, Hl * d, h, r * Hl * d, 0, bq);
          w->go = falloc(h * (Hl * d / 128));
          gen_shard_i8_groups(w->qo, w->go, h, Hl * d, h, h, h, 0, r * Hl * d, bo);
          w->gup = falloc(Fl * (h / 128));
          gen_shard_i8_groups(w->qup, w->gup, Fl, h, h, Fl, m->F, r * Fl, 0, bu);
          w->gdown = falloc(h * (Fl / 128));
          gen_shard_i8_groups(w->qdown, w->gdown, h, Fl, m->F, h, h, 0, r * Fl, bd);
        }
      }
    }
    ly->bqkv = falloc(3 * h);
    gen_vec(ly->bqkv, 3 * h, or_synth_base(seed, li, T_QKV_B), 0.f, kAmpB);
    ly->bo = falloc(h);
    gen_vec(ly->bo, h, or_synth_base(seed, li, T_O_B), 0.f, kAmpB);
    ly->bup = falloc(m->F);
    gen_vec(ly->bup, m->F, or_synth_base(seed, li, T_UP_B), 0.f, kAmpB);
    ly->bdown = falloc(h);
    gen_vec(ly->bdown, h, or_synth_base(seed, li, T_DOWN_B), 0.f, kAmpB);
    ly->ln1g = falloc(h);
    gen_vec(ly->ln1g, h, or_synth_base(seed, li, T_LN1_G), 1.f, kAmpG);
    ly->ln1b = falloc(h);
    gen_vec(ly->ln1b, h, or_synth_base(seed, li, T_LN1_B), 0.f, kAmpBeta);
    ly->ln2g = falloc(h);
    gen_vec(ly->ln2g, h, or_synth_base(seed, li, T_LN2_G), 1.f, kAmpG);
    ly->ln2b = falloc(h);
    gen_vec(ly->ln2b, h, or_synth_base(seed, li, T_LN2_B), 0.f, kAmpBeta);
  }
  const uint64_t bw = or_synth_base(seed, -1, T_WTE);
  m->wte = falloc(m->V * h);
  gen_shard(m->wte, m->V, h, h, m->V, m->V, 0, 0, m->V, bw);
  m->wlm = (float**)calloc((size_t)m->t, sizeof(float*));
  for (int r = 0; r < m->t; ++r) {
    m->wlm[r] = falloc(m->Vl * h);
    gen_shard(m->wlm[r], m->Vl, h, h, m->Vl, m->Vpad, r * m->Vl, 0, m->V, bw);
  }
  m->lnfg = falloc(h);
  gen_vec(m->lnfg, h, or_synth_base(seed, -1, T_LNF_G), 1.f, kAmpG);
  m->lnfb = falloc(h);
  gen_vec(m->lnfb, h, or_synth_base(seed, -1, T_LNF_B), 0.f, kAmpBeta);
  /* rotary table: same expression as the device runtime's host-side table (model.cu) */
  m->rope = falloc(cfg->max_ctx * d);
  for (int64_t p = 0; p < cfg->max_ctx; ++p)
    for (int64_t i = 0; i < d / 2; ++i) {
      const double inv = pow((double)m->c.rope_base, -2.0 * (double)i / (double)d);
      const double ang = (double)p * inv;
      m->rope[(p * (d / 2) + i) * 2] = (float)cos(ang);
      m->rope[(p * (d / 2) + i) * 2 + 1] = (float)sin(ang);
    }
  const int64_t kv = m->L * m->B * m->H * cfg->max_ctx * d;
  m->kc = falloc(kv);
  m->vc = falloc(kv);
  m->res = falloc(m->B * h);
  m->final_hidden = falloc(m->B * h);
  return m;
}

void or_model_destroy(or_model* m) {
  if (!m) return;
  for (int64_t l = 0; l < m->L; ++l) {
    or_layer* ly = &m->layers[l];
    for (int r = 0; r < m->t; ++r) {
      or_rank_w* w = &ly->ranks[r];
      free(w->wqkv); free(w->wo); free(w->wup); free(w->wdown);
      free(w->qqkv); free(w->qo); free(w->qup); free(w->qdown);
      free(w->sqkv); free(w->so); free(w->sup); free(w->sdown);
      free(w->gqkv); free(w->go); free(w->gup); free(w->gdown);
    }
    free(ly->ranks);
    free(ly->bqkv); free(ly->bo); free(ly->bup); free(ly->bdown);
    free(ly->ln1g); free(ly->ln1b); free(ly->ln2g); free(ly->ln2b);
  }
  free(m->layers);
  for (int r = 0; r < m->t; ++r) free(m->wlm[r]);
  free(m->wlm);
  free(m->wte); free(m->lnfg); free(m->lnfb); free(m->rope);
  free(m->kc); free(m->vc); free(m->res); free(m->final_hidden);
  free(m);
}

/* LayerNorm in fp64 over an fp32 row, output rounded fp32 -> fp16 (the GPU's storage point). */
static void layernorm_row(const float* v, int64_t K, const float* g, const float* b, float eps, float* out16) {
  double mean = 0.0;
  for (int64_t k = 0; k < K; ++k) mean += v[k];
  mean /= (double)K;
  double var = 0.0;
  for (int64_t k = 0; k < K; ++k) var += (v[k] - mean) * (v[k] - mean);
  var /= (double)K;
  const double rstd = 1.0 / sqrt(var + (double)eps);
  for (int64_t k = 0; k < K; ++k) out16[k] = f16r((float)((v[k] - mean) * rstd * g[k] + b[k]));
}

static double gelu_tanh(double x) { return 0.5 * x * (1.0 + tanh(0.7978845608028654 * (x + 0.044715 * x * x * x))); }

/* fp16 path GEMM: out[b][n] (double) over the rank's row-major shard with the rank's schedule */
static or_gemm_hook_fn g_hook;
static void* g_hook_ctx;
static void gemm16(const float* W, int64_t N, int64_t K, int sm, const float* x16, int64_t B, double* out) {
  or_schedule s;
  or_derive_schedule(N, K, B, 2, sm, &s);
  double* xd = (double*)malloc(sizeof(double) * (size_t)(B * K));
  for (int64_t i = 0; i < B * K; ++i) xd[i] = x16[i];
  if (g_hook) g_hook(W, N, K, xd, B, out, g_hook_ctx);
  else or_gemm_f64(W, N, K, &s, xd, B, out);
  free(xd);
}

/* int8 weights, fp16 activations (W8A16, weight-only): y = fp32(sum_k q w_k x_k) * s_w (the sum in
 * fp64 here; the GPU accumulates the exact int8 x fp16 products in fp32) */
static void gemm8_a16(const int8_t* W, const float* ws, int64_t N, int64_t K, const float* x16, int64_t B, float* y) {
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < N; ++n)
    for (int64_t b = 0; b < B; ++b) {
      double a = 0.0;
      for (int64_t k = 0; k < K; ++k) a += (double)W[n * K + k] * (double)x16[b * K + k];
      y[b * N + n] = (float)a * ws[n];
    }
}

/* Activation mode of layer GEMM g (0 QKV, 1 attn-out, 2 MLP-up, 3 MLP-down). */
static int act_of(int int8_act, int g) { return (int8_act & 0x100) ? (int8_act >> g) & 1 : int8_act; }

/* int8 path GEMM on fp16 activations: per-token quantisation, exact int32, fp32 dequant
 * (int8_act 1: weight-only, fp16 activations) */
static void gemm8(int int8_act, const int8_t* W, const float* ws, int64_t N, int64_t K, const float* x16, int64_t B,
                  float* y, const float* gs) {
  if (gs != NULL) { /* K-group weight-only: y = sum_g s_g sum_{k in g} q x (fp64; the GPU: fp32 per group) */
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; ++n)
      for (int64_t b = 0; b < B; ++b) {
        double a = 0.0;
        for (int64_t k = 0; k < K; ++k) a += (double)W[n * K + k] * (double)gs[(k / 128) * N + n] * (double)x16[b * K + k];
        y[b * N + n] = (float)a;
      }
    return;
  }
  if (int8_act == 1) {
    gemm8_a16(W, ws, N, K, x16, B, y);
    return;
  }
  int8_t* xq = (int8_t*)malloc((size_t)(B * K));
  float* xs = falloc(B);
  or_quant_rows(x16, B, K, xq, xs);
  or_gemm_i8(W, ws, xq, xs, N, K, B, NULL, y);
  free(xq);
  free(xs);
}

int or_model_step(or_model* m, const int32_t* tokens, int64_t pos, float* logits, int32_t* next_tokens) {
  const int64_t h = m->h, d = m->d, Hl = m->Hl, B = m->B, Fl = m->Fl, mc = m->c.max_ctx;
  const int i8 = m->c.dtype_bytes == 1;
  const int sm = m->c.sm_count;
  if (pos < 0 || pos >= mc) return 2;
  g_hook = m->hook;
  g_hook_ctx = m->hook_ctx;
  float* r = m->res;
  for (int64_t b = 0; b < B; ++b) {
    int32_t tok = tokens[b];
    if (tok < 0 || tok >= m->V) tok = 0;
    memcpy(r + b * h, m->wte + tok * h, sizeof(float) * (size_t)h);
  }
  float* xln = falloc(B * h);
  float* dsum = falloc(B * h);
  float* a16 = falloc(B * h);
  float* u16 = falloc(B * Fl);
  int64_t maxn = 3 * h;
  if (m->F > maxn) maxn = m->F;
  if (m->Vl > maxn) maxn = m->Vl;
  double* yd = (double*)malloc(sizeof(double) * (size_t)(B * maxn));
  float* yf = falloc(B * maxn);
  const double scale = 1.0 / sqrt((double)d);
  for (int64_t l = 0; l < m->L; ++l) {
    or_layer* ly = &m->layers[l];
    if (l > 0) { /* residual += d_mlp + b_down (fp32, in the GPU's order) */
      const float* bd = m->layers[l - 1].bdown;
      for (int64_t b = 0; b < B; ++b)
        for (int64_t k = 0; k < h; ++k) {
          const float t = dsum[b * h + k] + bd[k];
          r[b * h + k] = r[b * h + k] + t;
        }
    }
    for (int64_t b = 0; b < B; ++b) layernorm_row(r + b * h, h, ly->ln1g, ly->ln1b, m->c.ln_eps, xln + b * h);
    memset(dsum, 0, sizeof(float) * (size_t)(B * h));
    for (int rk = 0; rk < m->t; ++rk) {
      or_rank_w* w = &ly->ranks[rk];
      const int64_t Nq = 3 * Hl * d;
      /* K1: QKV + bias + RoPE + KV append */
      if (!i8) gemm16(w->wqkv, Nq, h, sm, xln, B, yd);
      else gemm8(act_of(m->c.int8_act, 0), w->qqkv, w->sqkv, Nq, h, xln, B, yf, w->gqkv);
      for (int64_t b = 0; b < B; ++b)
        for (int64_t n = 0; n < Nq; n += 2) {
          const int64_t sec = n / (Hl * d), rem = n % (Hl * d), hh = rem / d, i = rem % d;
          const int64_t gn = sec * h + rk * Hl * d + rem;
          float o0, o1;
          const float c = m->rope[(pos * (d / 2) + i / 2) * 2], s = m->rope[(pos * (d / 2) + i / 2) * 2 + 1];
          if (!i8) {
            double y0 = yd[b * Nq + n] + ly->bqkv[gn], y1 = yd[b * Nq + n + 1] + ly->bqkv[gn + 1];
            if (sec < 2) {
              const double r0 = y0 * c - y1 * s, r1 = y0 * s + y1 * c;
              y0 = r0;
              y1 = r1;
            }
            o0 = f16r((float)y0);
            o1 = f16r((float)y1);
          } else { /* fp32 ops in the device epilogue's order */
            float y0 = yf[b * Nq + n] + ly->bqkv[gn], y1 = yf[b * Nq + n + 1] + ly->bqkv[gn + 1];
            if (sec < 2) {
              const float p0 = y0 * c, p1 = y1 * s, p2 = y0 * s, p3 = y1 * c;
              y0 = p0 - p1;
              y1 = p2 + p3;
            }
            o0 = f16r(y0);
            o1 = f16r(y1);
          }
          const int64_t ghead = rk * Hl + hh;
          if (sec == 0) {
            /* stash q in the a16 buffer temporarily: [B][H*d] global head order */
            a16[b * h + ghead * d + i] = o0;
            a16[b * h + ghead * d + i + 1] = o1;
          } else {
            float* cache = sec == 1 ? m->kc : m->vc;
            const int64_t off = ((((l * B + b) * m->H + ghead) * mc) + pos) * d + i;
            cache[off] = o0;
            cache[off + 1] = o1;
          }
        }
    }
    /* K2: attention per (b, head), fp64 softmax; q is in a16, output overwrites it per head */
    {
      double* sc = (double*)malloc(sizeof(double) * (size_t)(pos + 1));
      double* o = (double*)malloc(sizeof(double) * (size_t)d);
      for (int64_t b = 0; b < B; ++b)
        for (int64_t hh = 0; hh < m->H; ++hh) {
          const float* q = a16 + b * h + hh * d;
          const float* kb = m->kc + ((l * B + b) * m->H + hh) * mc * d;
          const float* vb = m->vc + ((l * B + b) * m->H + hh) * mc * d;
          double mx = -INFINITY;
          for (int64_t j = 0; j <= pos; ++j) {
            double acc = 0.0;
            for (int64_t i = 0; i < d; ++i) acc += (double)q[i] * (double)kb[j * d + i];
            sc[j] = acc * scale;
            if (sc[j] > mx) mx = sc[j];
          }
          double l_sum = 0.0;
          for (int64_t j = 0; j <= pos; ++j) {
            sc[j] = exp(sc[j] - mx);
            l_sum += sc[j];
          }
          for (int64_t i = 0; i < d; ++i) o[i] = 0.0;
          for (int64_t j = 0; j <= pos; ++j)
            for (int64_t i = 0; i < d; ++i) o[i] += sc[j] * (double)vb[j * d + i];
          float* dst = a16 + b * h + hh * d;
          for (int64_t i = 0; i < d; ++i) dst[i] = f16r((float)(o[i] / l_sum));
        }
      free(sc);
      free(o);
    }
    /* K3: attn-out (row parallel) -> fp32 partials summed in rank order */
    for (int rk = 0; rk < m->t; ++rk) {
      or_rank_w* w = &ly->ranks[rk];
      float* xa = falloc(B * Hl * d);
      for (int64_t b = 0; b < B; ++b) memcpy(xa + b * Hl * d, a16 + b * h + rk * Hl * d, sizeof(float) * (size_t)(Hl * d));
      if (!i8) {
        gemm16(w->wo, h, Hl * d, sm, xa, B, yd);
        for (int64_t i = 0; i < B * h; ++i) yf[i] = (float)yd[i];
      } else {
        gemm8(act_of(m->c.int8_act, 1), w->qo, w->so, h, Hl * d, xa, B, yf, w->go);
      }
      for (int64_t i = 0; i < B * h; ++i) dsum[i] = rk == 0 ? yf[i] : dsum[i] + yf[i];
      free(xa);
    }
    /* K4 prologue: residual += d_attn + b_o ; LN2 */
    for (int64_t b = 0; b < B; ++b)
      for (int64_t k = 0; k < h; ++k) {
        const float t = dsum[b * h + k] + ly->bo[k];
        r[b * h + k] = r[b * h + k] + t;
      }
    for (int64_t b = 0; b < B; ++b) layernorm_row(r + b * h, h, ly->ln2g, ly->ln2b, m->c.ln_eps, xln + b * h);
    float* dm = falloc(B * h);
    for (int rk = 0; rk < m->t; ++rk) {
      or_rank_w* w = &ly->ranks[rk];
      /* K4: up + bias + GeLU (column parallel) */
      if (!i8) {
        gemm16(w->wup, Fl, h, sm, xln, B, yd);
        for (int64_t b = 0; b < B; ++b)
          for (int64_t n = 0; n < Fl; ++n)
            u16[b * Fl + n] = f16r((float)gelu_tanh(yd[b * Fl + n] + ly->bup[rk * Fl + n]));
      } else {
        gemm8(act_of(m->c.int8_act, 2), w->qup, w->sup, Fl, h, xln, B, yf, w->gup);
        for (int64_t b = 0; b < B; ++b)
          for (int64_t n = 0; n < Fl; ++n) {
            const float y = yf[b * Fl + n] + ly->bup[rk * Fl + n];
            u16[b * Fl + n] = f16r((float)gelu_tanh((double)y));
          }
      }
      /* K5: down (row parallel) */
      if (!i8) {
        gemm16(w->wdown, h, Fl, sm, u16, B, yd);
        for (int64_t i = 0; i < B * h; ++i) yf[i] = (float)yd[i];
      } else {
        gemm8(act_of(m->c.int8_act, 3), w->qdown, w->sdown, h, Fl, u16, B, yf, w->gdown);
      }
      for (int64_t i = 0; i < B * h; ++i) dm[i] = rk == 0 ? yf[i] : dm[i] + yf[i];
    }
    memcpy(dsum, dm, sizeof(float) * (size_t)(B * h));
    free(dm);
  }
  /* final: residual + d_mlp + b_down ; final LN ; LM head (fp16, vocab parallel) ; argmax */
  if (m->L > 0) {
    const float* bd = m->layers[m->L - 1].bdown;
    for (int64_t b = 0; b < B; ++b)
      for (int64_t k = 0; k < h; ++k) {
        const float t = dsum[b * h + k] + bd[k];
        r[b * h + k] = r[b * h + k] + t;
      }
  }
  for (int64_t b = 0; b < B; ++b) layernorm_row(r + b * h, h, m->lnfg, m->lnfb, m->c.ln_eps, xln + b * h);
  memcpy(m->final_hidden, xln, sizeof(float) * (size_t)(B * h));
  for (int rk = 0; rk < m->t; ++rk) {
    gemm16(m->wlm[rk], m->Vl, h, sm, xln, B, yd);
    for (int64_t b = 0; b < B; ++b)
      for (int64_t n = 0; n < m->Vl; ++n) {
        const int64_t g = rk * m->Vl + n;
        if (g < m->V) logits[b * m->V + g] = (float)yd[b * m->Vl + n];
      }
  }
  for (int64_t b = 0; b < B; ++b) {
    int32_t best = 0;
    for (int64_t v = 1; v < m->V; ++v)
      if (logits[b * m->V + v] > logits[b * m->V + best]) best = (int32_t)v;
    if (next_tokens) next_tokens[b] = best;
  }
  free(xln);
  free(dsum);
  free(a16);
  free(u16);
  free(yd);
  free(yf);
  return 0;
}

void or_model_final_hidden(const or_model* m, float* out) {
  memcpy(out, m->final_hidden, sizeof(float) * (size_t)(m->B * m->h));
}
