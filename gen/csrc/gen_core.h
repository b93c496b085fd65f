/*
 * gen_core.h — seeded, counter-based synthetic trace generator (TEST/BENCH INPUT ONLY).
 *
 * This header holds NONE of the method's arithmetic (no interning, no tree building, no
 * aggregation). It only draws synthetic inputs: per-record site choice, path length,
 * frames, metrics and PC samples, from a stateless counter hash so that the host loop
 * (used to feed the CPU oracle) and the device kernel (used to feed the CUDA path) emit
 * byte-identical traces by construction. Program tables (sites, their frame paths,
 * per-site base times, per-kernel PC/stall CDFs) are built once on the host in Python
 * (gen/programs.py) and passed in as plain arrays.
 *
 * Recipe: DESIGN.md "Input recipe" and SURVEY.md §8(d) "Generator rules".
 */
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define GEN_HD __host__ __device__ __forceinline__
#else
#define GEN_HD static inline
#endif

/* stream tags */
enum {
  GS_SITE = 1, GS_TRUNC = 2, GS_TRUNCLEN = 3, GS_REC = 4, GS_RECPOS = 5, GS_NSE = 6,
  GS_NS = 7, GS_CNT = 8, GS_JIT = 9, GS_BLK = 10, GS_DYN = 11, GS_DYNLEN = 12,
  GS_PC = 13, GS_STALL = 14, GS_LEN = 15, GS_BAD = 16, GS_BADKIND = 17
};

GEN_HD uint64_t gen_mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27; z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}
GEN_HD uint64_t gen_rnd(uint64_t seed, uint64_t stream, uint64_t i) {
  return gen_mix64(seed ^ (stream * 0x9E3779B97F4A7C15ull) ^ (i * 0xD1B54A32D192ED03ull));
}

typedef struct { uint32_t kind, str_id; uint64_t addr; } gen_key; /* 16 B, same layout as dc_frame_key */

enum { GEN_SEQ = 0, GEN_RANDOM = 1 };
enum { GEN_MET_CFG1 = 1, GEN_MET_CFG2 = 2, GEN_MET_NS_COUNT = 3 };

typedef struct {
  uint64_t seed;
  uint32_t mode;          /* GEN_SEQ: site = r mod n_sites; GEN_RANDOM: site = rnd % n_sites */
  uint32_t n_sites;
  const uint32_t* site_off;     /* [n_sites+1] offsets into site_frames */
  const uint32_t* site_frames;  /* pool indices */
  /* GEN_RANDOM extras (config 1) */
  uint32_t trunc_permille;      /* records ending at an interior node */
  uint32_t rec_permille;        /* records with an A->A->A recursive segment */
  uint32_t max_depth;           /* recursion insertion skipped if it would exceed this */
  uint32_t empty_mod, empty_rem;/* r % empty_mod == empty_rem -> empty path (empty_mod 0: none) */
  uint64_t force_record;        /* record force_record takes site force_site whole */
  uint32_t force_site;
  /* GEN_SEQ recursion (config 4): k frames alternating rec_a, rec_b inserted at rec_pos */
  const uint32_t* site_rec_k;   /* [n_sites] or NULL */
  uint32_t rec_pos, rec_a, rec_b;
  uint32_t dyn_per100k;         /* records drawing a per-record total depth */
  uint32_t dyn_min, dyn_max;
  /* metrics */
  uint32_t met_kind, n_metrics;
  const uint64_t* site_base_ns; /* [n_sites] */
  const uint32_t* site_warps;   /* [n_sites] */
  const uint32_t* site_smem;    /* [n_sites] */
} gen_prog;

/* Per-record shape: site, base length, truncated length and recursion insertion. */
typedef struct { uint32_t site, base_len, len, ins_pos, ins_k, ins_kind; } gen_shape;
/* ins_kind 0: none; 1: repeat frame at ins_pos ins_k more times; 2: alternate rec_a/rec_b */

GEN_HD gen_shape gen_record_shape(const gen_prog* p, uint64_t r) {
  gen_shape s; s.ins_pos = 0; s.ins_k = 0; s.ins_kind = 0;
  if (p->mode == GEN_RANDOM) {
    if (p->empty_mod && (r % p->empty_mod) == p->empty_rem) {
      s.site = 0; s.base_len = 0; s.len = 0; return s;
    }
    int forced = (r == p->force_record);
    s.site = forced ? p->force_site : (uint32_t)(gen_rnd(p->seed, GS_SITE, r) % p->n_sites);
    s.base_len = p->site_off[s.site + 1] - p->site_off[s.site];
    s.len = s.base_len;
    if (!forced && s.len > 1 && (gen_rnd(p->seed, GS_TRUNC, r) % 1000) < p->trunc_permille)
      s.len = 1 + (uint32_t)(gen_rnd(p->seed, GS_TRUNCLEN, r) % s.len);
    if (!forced && s.len >= 1 && s.len + 2 <= p->max_depth &&
        (gen_rnd(p->seed, GS_REC, r) % 1000) < p->rec_permille) {
      s.ins_kind = 1; s.ins_k = 2;
      s.ins_pos = (uint32_t)(gen_rnd(p->seed, GS_RECPOS, r) % s.len);
      s.len += 2;
    }
    return s;
  }
  s.site = (uint32_t)(r % p->n_sites);
  s.base_len = p->site_off[s.site + 1] - p->site_off[s.site];
  s.len = s.base_len;
  uint32_t k = p->site_rec_k ? p->site_rec_k[s.site] : 0;
  if (p->dyn_per100k && (gen_rnd(p->seed, GS_DYN, r) % 100000) < p->dyn_per100k) {
    uint32_t span = p->dyn_max - p->dyn_min + 1;
    uint32_t target = p->dyn_min + (uint32_t)(gen_rnd(p->seed, GS_DYNLEN, r) % span);
    k = target > s.base_len ? target - s.base_len : 0;
  }
  if (k && s.base_len >= p->rec_pos) {
    s.ins_kind = 2; s.ins_k = k; s.ins_pos = p->rec_pos; s.len += k;
  }
  return s;
}

/* Pool index of frame j (0 <= j < s.len) of a record with shape s. */
GEN_HD uint32_t gen_record_frame(const gen_prog* p, const gen_shape* s, uint32_t j) {
  const uint32_t* f = p->site_frames + p->site_off[s->site];
  if (s->ins_kind == 1) {
    if (j <= s->ins_pos) return f[j];
    if (j <= s->ins_pos + s->ins_k) return f[s->ins_pos];
    return f[j - s->ins_k];
  }
  if (s->ins_kind == 2) {
    if (j < s->ins_pos) return f[j];
    if (j < s->ins_pos + s->ins_k) return ((j - s->ins_pos) & 1) ? p->rec_b : p->rec_a;
    return f[j - s->ins_k];
  }
  return f[j];
}

GEN_HD uint64_t gen_pow10(uint32_t e) { uint64_t v = 1; while (e--) v *= 10; return v; }

/* Metric m of record r (integer draws only). */
GEN_HD uint64_t gen_record_metric(const gen_prog* p, const gen_shape* s, uint64_t r, uint32_t m) {
  if (p->met_kind == GEN_MET_CFG1) {
    if (m == 0) {
      if (r % 1000 == 5) return 0;
      if (r % 1000 == 6) return 1ull << 40;
      uint32_t e = 1 + (uint32_t)(gen_rnd(p->seed, GS_NSE, r) % 9);
      return 1 + gen_rnd(p->seed, GS_NS, r) % gen_pow10(e);
    }
    return 1 + gen_rnd(p->seed, GS_CNT, r) % 4;
  }
  uint64_t base = p->site_base_ns[s->site];
  if (m == 0) return base * (950 + gen_rnd(p->seed, GS_JIT, r) % 101) / 1000;
  if (m == 1) return 1;
  if (p->met_kind == GEN_MET_CFG2) {
    if (m == 2) return 1ull << (gen_rnd(p->seed, GS_BLK, r) % 17);
    if (m == 3) return p->site_warps[s->site];
    return p->site_smem[s->site];
  }
  return 0;
}

/* ---- PC samples (config 3): contiguous runs per launch ------------------------------ */
typedef struct { uint32_t launch, pc_off; uint16_t stall, flags; uint32_t count; } gen_pc_sample;

typedef struct {
  uint64_t seed;
  uint32_t n_launch, n_sites;        /* launch l runs the kernel of site l mod n_sites */
  const uint64_t* launch_off;        /* [n_launch+1] */
  const uint32_t* site_kernel;       /* [n_sites] kernel type of each site */
  const uint32_t* kern_off;          /* [n_kern+1] offsets into pc tables */
  const uint32_t* pc_thr;            /* per kernel: n_pc entries; entry j<n_pc-1 = upper CDF bound (31-bit) */
  const uint32_t* pc_instr;          /* per kernel rank -> instruction index */
  const uint32_t* stall_thr;         /* [total_pc*3] 31-bit thresholds, 0xFFFFFFFF = unused */
  const uint8_t*  stall_id;          /* [total_pc*4] */
  uint32_t n_stall;
  uint32_t bad_per_million;          /* inject invalid samples (tests only) */
} gen_pc_prog;

GEN_HD gen_pc_sample gen_pc_draw(const gen_pc_prog* q, uint32_t l, uint64_t i) {
  gen_pc_sample o;
  uint32_t k = q->site_kernel[l % q->n_sites];
  uint32_t b = q->kern_off[k], n = q->kern_off[k + 1] - b;
  uint32_t u = (uint32_t)(gen_rnd(q->seed, GS_PC, i) >> 33);
  /* j = number of thresholds <= u among the first n-1 (upper-bound binary search) */
  uint32_t lo = 0, hi = n - 1;
  while (lo < hi) { uint32_t mid = (lo + hi) >> 1; if (q->pc_thr[b + mid] <= u) lo = mid + 1; else hi = mid; }
  uint32_t g = b + lo;
  uint32_t u2 = (uint32_t)(gen_rnd(q->seed, GS_STALL, i) >> 33);
  uint32_t c = 0;
  while (c < 3 && q->stall_thr[(uint64_t)g * 3 + c] <= u2) ++c;
  o.launch = l;
  o.pc_off = 16u * q->pc_instr[g];
  o.stall = q->stall_id[(uint64_t)g * 4 + c];
  o.flags = 0;
  o.count = 1;
  if (q->bad_per_million && (gen_rnd(q->seed, GS_BAD, i) % 1000000) < q->bad_per_million) {
    uint32_t t = (uint32_t)(gen_rnd(q->seed, GS_BADKIND, i) % 3);
    if (t == 0) o.launch = q->n_launch + (uint32_t)(i % 7);
    else if (t == 1) o.stall = (uint16_t)(q->n_stall + (i % 5));
    else o.count = 0;
  }
  return o;
}
