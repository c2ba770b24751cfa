/* TEST INFRASTRUCTURE ONLY -- plain-C restatement of the HyperOMS (`homs`) hot path.
 *
 * See homs_oracle.h for the usage rule (checker only, never on the product path) and for the
 * parity status (PINNED against the reference's known answers, SURVEY.md 8(c) fingerprints and
 * the compiled reference in oracle/_ref/).
 *
 * Every function cites the reference lines (under /root/reference/proj/core/) it restates.
 * Written for clarity, not speed: scalar loops, one thread.
 */
#define _GNU_SOURCE
#include "homs_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_error[256];

static long long fail(const char* kind, const char* msg) {
  snprintf(g_error, sizeof g_error, "%s: %s", kind, msg);
  return -1;
}

const char* ho_last_error(void) { return g_error; }

/* FNV-1a 64 exactly as src/cache.cpp:18-29 has it.  NOTE the reference seeds the state with
 * 1469598103934665603 (not the textbook basis 14695981039346656037); fingerprints in
 * SURVEY.md 8(c) were taken with the reference constant, so it is restated verbatim. */
uint64_t ho_fnv1a64(const void* data, uint64_t n_bytes) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 1469598103934665603ULL;
  for (uint64_t i = 0; i < n_bytes; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* ---- RNG: std::mt19937_64 (ISO C++ [rand.predef]) + include/homs/rng.hpp ------------------ */

#define MT_N 312
#define MT_M 156
typedef struct {
  uint64_t mt[MT_N];
  int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = MT_N;
}

static uint64_t mt64_next(mt64* s) {
  if (s->idx >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % MT_N] & 0x7FFFFFFFULL);
      s->mt[i] = s->mt[(i + MT_M) % MT_N] ^ (x >> 1) ^ ((x & 1) ? 0xB5026F5AA96619E9ULL : 0);
    }
    s->idx = 0;
  }
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* rng.hpp:10-15 */
static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
/* rng.hpp:19-21 */
static uint64_t stream_seed(uint64_t seed, uint64_t tag) {
  return splitmix64(seed ^ splitmix64(tag));
}
/* rng.hpp:26-39: mask rejection */
static uint64_t bounded_uniform(mt64* rng, uint64_t n) {
  uint64_t mask = n - 1;
  mask |= mask >> 1;
  mask |= mask >> 2;
  mask |= mask >> 4;
  mask |= mask >> 8;
  mask |= mask >> 16;
  mask |= mask >> 32;
  uint64_t v;
  do {
    v = mt64_next(rng) & mask;
  } while (v >= n);
  return v;
}
/* rng.hpp:42-44 */
static double uniform_unit(mt64* rng) { return (double)(mt64_next(rng) >> 11) * 0x1.0p-53; }

/* ---- hypervector helpers: include/homs/hypervector.hpp ------------------------------------ */

static size_t words_for(uint32_t bits) { return ((size_t)bits + 63) / 64; } /* :26-28 */

static void mask_tail(uint64_t* w, uint32_t bits) { /* :45-49 */
  if (bits % 64 != 0 && bits != 0) w[words_for(bits) - 1] &= (((uint64_t)1) << (bits % 64)) - 1;
}
static void flip_bit(uint64_t* w, uint32_t i) { w[i / 64] ^= ((uint64_t)1) << (i % 64); }
static int get_bit(const uint64_t* w, uint32_t i) { return (int)((w[i / 64] >> (i % 64)) & 1u); }

static uint32_t popcount64(uint64_t x) { /* std::popcount, done the slow portable way */
  uint32_t n = 0;
  while (x) {
    x &= x - 1;
    ++n;
  }
  return n;
}

/* hypervector.hpp:70-81 (packed) and tests/oracles.hpp:26-33 (per bit) */
long long ho_hamming_similarity(uint32_t dim, const uint64_t* a, const uint64_t* b, int bitwise) {
  if (bitwise) {
    uint32_t same = 0;
    for (uint32_t d = 0; d < dim; ++d) same += get_bit(a, d) == get_bit(b, d);
    return same;
  }
  uint32_t diff = 0;
  for (size_t i = 0; i < words_for(dim); ++i) diff += popcount64(a[i] ^ b[i]);
  return (long long)dim - diff;
}

/* ---- preprocess: src/preprocess.cpp ------------------------------------------------------- */

static const double kBinEpsilon = 1e-9; /* :17 */

long long ho_validate_preprocess(const ho_precfg* c) { /* :21-34 */
  if (!(c->min_mz < c->max_mz)) return fail("ConfigError", "min_mz must be smaller than max_mz");
  if (!(c->bin_size > 0.0)) return fail("ConfigError", "bin_size must be positive");
  if (c->min_peaks < 1 || c->max_peaks < c->min_peaks)
    return fail("ConfigError", "need max_peaks >= min_peaks >= 1");
  if (!(c->intensity_floor >= 0.0 && c->intensity_floor < 1.0))
    return fail("ConfigError", "intensity_floor must lie in [0, 1)");
  return 0;
}

long long ho_dimension(const ho_precfg* c) { /* :36-39 */
  const double q = (c->max_mz - c->min_mz) / c->bin_size;
  return (uint32_t)ceil(q - kBinEpsilon);
}

typedef struct {
  double mz, intensity;
} peak;

static int cmp_intensity_desc_mz_asc(const void* x, const void* y) { /* :60-63 */
  const peak *a = x, *b = y;
  if (a->intensity != b->intensity) return a->intensity > b->intensity ? -1 : 1;
  if (a->mz != b->mz) return a->mz < b->mz ? -1 : 1;
  return 0;
}
static int cmp_mz_asc(const void* x, const void* y) { /* :65-66 */
  const peak *a = x, *b = y;
  if (a->mz != b->mz) return a->mz < b->mz ? -1 : 1;
  return 0;
}

/* refine_peaks :41-75.  Writes survivors to `kept`, returns their count or -1 for nullopt.
 * NOTE: like the reference, correct only for the RawSpectrum invariant "peaks strictly
 * ascending in m/z" (include/homs/spectrum.hpp:34-35); with duplicate m/z the reference's
 * second std::sort leaves their relative order unspecified. */
static long long refine_peaks(const ho_precfg* c, uint64_t n, const double* mz,
                              const double* inten, peak* kept) {
  size_t m = 0;
  for (uint64_t i = 0; i < n; ++i) /* :45-49 */
    if (mz[i] >= c->min_mz && mz[i] < c->max_mz && inten[i] > 0.0) {
      kept[m].mz = mz[i];
      kept[m].intensity = inten[i];
      ++m;
    }
  if (m > 0) { /* :51-56 */
    double base = 0.0;
    for (size_t i = 0; i < m; ++i) base = base < kept[i].intensity ? kept[i].intensity : base;
    const double floor_intensity = c->intensity_floor * base;
    size_t w = 0;
    for (size_t i = 0; i < m; ++i)
      if (!(kept[i].intensity < floor_intensity)) kept[w++] = kept[i];
    m = w;
  }
  if (m > c->max_peaks) { /* :58-67 */
    qsort(kept, m, sizeof(peak), cmp_intensity_desc_mz_asc);
    m = c->max_peaks;
    qsort(kept, m, sizeof(peak), cmp_mz_asc);
  }
  if (m < c->min_peaks) return -1; /* :69 */
  return (long long)m;
}

/* vectorize :77-110 on refined peaks; returns number of bins */
static size_t vectorize(const ho_precfg* c, const peak* p, size_t m, uint32_t* bins,
                        double* vals) {
  const uint32_t dims = (uint32_t)ho_dimension(c);
  size_t nb = 0;
  for (size_t i = 0; i < m; ++i) { /* :91-101 */
    const double q = (p[i].mz - c->min_mz) / c->bin_size + kBinEpsilon;
    double f = floor(q);
    const double hi = (double)(dims - 1);
    if (f < 0.0) f = 0.0; /* std::clamp(v, lo, hi) */
    else if (hi < f) f = hi;
    const uint32_t bin = (uint32_t)f;
    if (nb > 0 && bins[nb - 1] == bin) {
      vals[nb - 1] += p[i].intensity;
    } else {
      bins[nb] = bin;
      vals[nb] = p[i].intensity;
      ++nb;
    }
  }
  if (c->scaling == 1) /* :103-105 */
    for (size_t k = 0; k < nb; ++k) vals[k] = sqrt(vals[k]);
  double top = vals[0]; /* :107-108 */
  for (size_t k = 1; k < nb; ++k) top = top < vals[k] ? vals[k] : top;
  for (size_t k = 0; k < nb; ++k) vals[k] /= top;
  return nb;
}

/* src/encoder.cpp:11-17 */
long long ho_quantize_intensity(double v, uint32_t levels) {
  if (!(v >= 0.0 && v <= 1.0)) return fail("InvariantError", "intensity outside [0, 1]");
  const double level = round(v * (double)levels);
  const uint32_t l = (uint32_t)level;
  return l < levels ? l : levels;
}

long long ho_refine_vectorize(const ho_precfg* cfg, uint64_t n_peaks, const double* mz,
                              const double* inten, uint32_t levels, uint32_t* out_bins,
                              double* out_intens, uint32_t* out_levels) {
  peak* kept = malloc((n_peaks + 1) * sizeof(peak));
  long long m = refine_peaks(cfg, n_peaks, mz, inten, kept);
  long long nb = 0;
  if (m > 0) {
    nb = (long long)vectorize(cfg, kept, (size_t)m, out_bins, out_intens);
    if (out_levels)
      for (long long k = 0; k < nb; ++k)
        out_levels[k] = (uint32_t)ho_quantize_intensity(out_intens[k], levels);
  } else if (m == 0) {
    /* min_peaks == 0 is rejected by validate(); vectorize would throw on an empty list */
    free(kept);
    return fail("InvariantError", "vectorize: refined spectrum has no peaks");
  }
  free(kept);
  return m < 0 ? 0 : nb;
}

/* ---- codebook: src/codebook.cpp ------------------------------------------------------------ */

typedef struct {
  uint32_t dim, step_flips, levels, n_bins;
  uint64_t seed;
  size_t W;
  uint64_t* pos; /* n_bins x W */
  uint64_t* lvl; /* (levels+1) x W */
} codebook;

static void random_hv(uint64_t* w, uint32_t dim, mt64* rng) { /* :17-22 */
  for (size_t i = 0; i < words_for(dim); ++i) w[i] = mt64_next(rng);
  mask_tail(w, dim);
}

void* ho_codebook_create(uint32_t dim, uint32_t step_flips, uint32_t levels, uint64_t seed,
                         uint32_t n_bins) {
  /* EncoderConfig::validate :26-36 is NOT called by make_codebook (:87-94); mirror that. */
  codebook* cb = calloc(1, sizeof *cb);
  cb->dim = dim;
  cb->step_flips = step_flips;
  cb->levels = levels;
  cb->n_bins = n_bins;
  cb->seed = seed;
  cb->W = words_for(dim);
  const size_t W = cb->W;
  cb->pos = calloc((size_t)(n_bins ? n_bins : 1) * W, 8);
  cb->lvl = calloc((size_t)(levels + 1) * W, 8);

  /* gen_position_hvs :38-53: chain of with-replacement flips */
  mt64 rng;
  mt64_seed(&rng, stream_seed(seed, 0x706f736974696f6eULL)); /* "position" :14 */
  uint64_t* cur = calloc(W, 8);
  random_hv(cur, dim, &rng); /* drawn even when n_bins == 0, as in the reference */
  if (n_bins > 0) memcpy(cb->pos, cur, W * 8);
  for (uint32_t i = 1; i < n_bins; ++i) {
    for (uint32_t k = 0; k < step_flips; ++k) flip_bit(cur, (uint32_t)bounded_uniform(&rng, dim));
    memcpy(cb->pos + (size_t)i * W, cur, W * 8);
  }

  /* gen_level_hvs :55-85: partial Fisher-Yates over dim positions, first dim/2 used */
  mt64_seed(&rng, stream_seed(seed, 0x6c6576656c687673ULL)); /* "levelhvs" :15 */
  const uint32_t flips_total = dim / 2;
  random_hv(cur, dim, &rng);
  uint32_t* order = malloc((size_t)dim * sizeof(uint32_t));
  for (uint32_t i = 0; i < dim; ++i) order[i] = i;
  for (uint32_t i = 0; i < flips_total; ++i) {
    const uint32_t j = i + (uint32_t)bounded_uniform(&rng, dim - i);
    const uint32_t t = order[i];
    order[i] = order[j];
    order[j] = t;
  }
  uint64_t flipped = 0;
  for (uint32_t q = 0; q <= levels; ++q) {
    const uint64_t cut = (uint64_t)flips_total * q / levels;
    for (; flipped < cut; ++flipped) flip_bit(cur, order[flipped]);
    memcpy(cb->lvl + (size_t)q * W, cur, W * 8);
  }
  free(order);
  free(cur);
  return cb;
}

void* ho_codebook_from_words(uint32_t dim, uint32_t levels, uint32_t n_bins, const uint64_t* pos,
                             const uint64_t* lvl) {
  codebook* cb = calloc(1, sizeof *cb);
  cb->dim = dim;
  cb->levels = levels;
  cb->n_bins = n_bins;
  cb->W = words_for(dim);
  cb->pos = malloc((size_t)n_bins * cb->W * 8);
  cb->lvl = malloc((size_t)(levels + 1) * cb->W * 8);
  memcpy(cb->pos, pos, (size_t)n_bins * cb->W * 8);
  memcpy(cb->lvl, lvl, (size_t)(levels + 1) * cb->W * 8);
  return cb;
}

void ho_codebook_export(const void* h, uint64_t* pos, uint64_t* lvl) {
  const codebook* cb = h;
  memcpy(pos, cb->pos, (size_t)cb->n_bins * cb->W * 8);
  memcpy(lvl, cb->lvl, (size_t)(cb->levels + 1) * cb->W * 8);
}

void ho_codebook_free(void* h) {
  codebook* cb = h;
  if (!cb) return;
  free(cb->pos);
  free(cb->lvl);
  free(cb);
}

/* ---- encode: src/encoder.cpp:19-55 ---------------------------------------------------------- */

static long long encode_sv(const codebook* cb, size_t nb, const uint32_t* bins, const double* vals,
                           int unpacked, uint64_t* out) {
  if (nb == 0) return fail("InvariantError", "encode: empty spectrum vector");
  const uint32_t dim = cb->dim;
  memset(out, 0, cb->W * 8);
  if (unpacked) { /* tests/oracles.hpp:36-55: bipolar accumulator, bit iff acc > 0 */
    long* acc = calloc(dim, sizeof(long));
    for (size_t k = 0; k < nb; ++k) {
      const long long lev = ho_quantize_intensity(vals[k], cb->levels);
      if (lev < 0) { free(acc); return -1; }
      const uint64_t* pw = cb->pos + (size_t)bins[k] * cb->W;
      const uint64_t* lw = cb->lvl + (size_t)lev * cb->W;
      for (uint32_t d = 0; d < dim; ++d)
        acc[d] += (get_bit(pw, d) ? 1 : -1) * (get_bit(lw, d) ? 1 : -1);
    }
    for (uint32_t d = 0; d < dim; ++d)
      if (acc[d] > 0) out[d / 64] |= ((uint64_t)1) << (d % 64);
    free(acc);
    return 0;
  }
  uint32_t* votes = calloc(dim, sizeof(uint32_t)); /* :33 */
  for (size_t k = 0; k < nb; ++k) {                /* :34-49 */
    if (bins[k] >= cb->n_bins) { free(votes); return fail("InvariantError", "bin out of range"); }
    const long long lev = ho_quantize_intensity(vals[k], cb->levels);
    if (lev < 0) { free(votes); return -1; }
    const uint64_t* pw = cb->pos + (size_t)bins[k] * cb->W;
    const uint64_t* lw = cb->lvl + (size_t)lev * cb->W;
    for (size_t w = 0; w < cb->W; ++w) {
      const uint64_t agree = ~(pw[w] ^ lw[w]);
      const uint32_t base = (uint32_t)w * 64;
      const uint32_t top = dim - base < 64 ? dim - base : 64;
      for (uint32_t b = 0; b < top; ++b) votes[base + b] += (uint32_t)((agree >> b) & 1u);
    }
  }
  for (uint32_t d = 0; d < dim; ++d) /* :51-53 strict majority, tie -> 0 */
    if (2ull * votes[d] > nb) out[d / 64] |= ((uint64_t)1) << (d % 64);
  free(votes);
  return 0;
}

long long ho_encode_vector(const void* codebook_h, uint32_t n_bins_sv, const uint32_t* bins,
                           const double* intens, int unpacked, uint64_t* out_words) {
  return encode_sv(codebook_h, n_bins_sv, bins, intens, unpacked, out_words);
}

/* src/pipeline.cpp:60-85 encode_spectra (threads/batch cannot change results; ignored) */
long long ho_encode_spectra(const void* codebook_h, const ho_precfg* cfg, uint64_t n,
                            const uint64_t* offsets, const double* mz, const double* inten,
                            unsigned threads, uint64_t batch, uint64_t* out_words,
                            uint8_t* out_ok) {
  (void)threads;
  (void)batch;
  const codebook* cb = codebook_h;
  if ((uint32_t)ho_dimension(cfg) != cb->n_bins) /* encoder.cpp:20-22 via sv.dims */
    return fail("InvariantError", "encode: spectrum vector dims do not match codebook");
  uint64_t max_p = 1;
  for (uint64_t i = 0; i < n; ++i)
    if (offsets[i + 1] - offsets[i] > max_p) max_p = offsets[i + 1] - offsets[i];
  peak* kept = malloc(max_p * sizeof(peak));
  uint32_t* bins = malloc(max_p * sizeof(uint32_t));
  double* vals = malloc(max_p * sizeof(double));
  long long unprocessable = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t* row = out_words + i * cb->W;
    memset(row, 0, cb->W * 8);
    out_ok[i] = 0;
    const uint64_t a = offsets[i], b = offsets[i + 1];
    const long long m = refine_peaks(cfg, b - a, mz + a, inten + a, kept);
    if (m < 0) { ++unprocessable; continue; }
    if (m == 0) { unprocessable = fail("InvariantError", "vectorize: no peaks"); break; }
    const size_t nb = vectorize(cfg, kept, (size_t)m, bins, vals);
    if (encode_sv(cb, nb, bins, vals, 0, row) < 0) { unprocessable = -1; break; }
    out_ok[i] = 1;
  }
  free(kept);
  free(bins);
  free(vals);
  return unprocessable;
}

/* ---- index: src/search.cpp:17-60 ------------------------------------------------------------ */

typedef struct {
  uint8_t charge;
  size_t n;
  double* mz;
  uint32_t* ordinal;
  uint64_t* words;
} bucket;

typedef struct {
  uint32_t dim;
  size_t W, n;
  /* metas in input order */
  double* mz;
  uint8_t* charge;
  uint8_t* is_decoy;
  char* id_blob;
  uint64_t* id_off;
  const uint64_t* words_in; /* copy of input rows (for linear search) */
  uint64_t* words_copy;
  size_t n_buckets;
  bucket* buckets; /* ascending charge (std::map order) */
} lib_index;

/* std::string operator< / == on ids: byte-wise unsigned compare, then length */
static int id_cmp(const lib_index* ix, uint32_t a, uint32_t b) {
  const size_t la = ix->id_off[a + 1] - ix->id_off[a], lb = ix->id_off[b + 1] - ix->id_off[b];
  const size_t m = la < lb ? la : lb;
  const int c = m ? memcmp(ix->id_blob + ix->id_off[a], ix->id_blob + ix->id_off[b], m) : 0;
  if (c != 0) return c;
  return la < lb ? -1 : (la > lb ? 1 : 0);
}

static int cmp_bucket_order(const void* x, const void* y, void* ctx) { /* :37-46 */
  const lib_index* ix = ctx;
  const uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
  if (ix->mz[a] != ix->mz[b]) return ix->mz[a] < ix->mz[b] ? -1 : 1;
  const int c = id_cmp(ix, a, b);
  if (c != 0) return c;
  return a < b ? -1 : (a > b ? 1 : 0);
}

void* ho_index_create(uint32_t dim, uint64_t n, const uint64_t* words, const double* mz,
                      const uint8_t* charge, const uint8_t* is_decoy, const char* id_blob,
                      const uint64_t* id_off) {
  if (n == 0) { fail("InvariantError", "build_index: library is empty"); return NULL; } /* :18 */
  lib_index* ix = calloc(1, sizeof *ix);
  ix->dim = dim;
  ix->W = words_for(dim);
  ix->n = n;
  ix->mz = malloc(n * 8);
  memcpy(ix->mz, mz, n * 8);
  ix->charge = malloc(n);
  memcpy(ix->charge, charge, n);
  ix->is_decoy = calloc(n, 1);
  if (is_decoy) memcpy(ix->is_decoy, is_decoy, n);
  ix->id_off = calloc(n + 1, 8);
  if (id_blob && id_off) {
    memcpy(ix->id_off, id_off, (n + 1) * 8);
    ix->id_blob = malloc(id_off[n] + 1);
    memcpy(ix->id_blob, id_blob, id_off[n]);
  } else {
    ix->id_blob = calloc(1, 1);
  }
  ix->words_copy = malloc(n * ix->W * 8);
  memcpy(ix->words_copy, words, n * ix->W * 8);
  ix->words_in = ix->words_copy;

  size_t count[256] = {0}; /* :30-33 group by charge */
  for (size_t i = 0; i < n; ++i) ++count[charge[i]];
  for (int c = 0; c < 256; ++c) ix->n_buckets += count[c] != 0;
  ix->buckets = calloc(ix->n_buckets, sizeof(bucket));
  size_t bi = 0;
  for (int c = 0; c < 256; ++c) {
    if (!count[c]) continue;
    bucket* b = &ix->buckets[bi++];
    b->charge = (uint8_t)c;
    b->n = count[c];
    b->ordinal = malloc(b->n * sizeof(uint32_t));
    size_t k = 0;
    for (size_t i = 0; i < n; ++i)
      if (charge[i] == c) b->ordinal[k++] = (uint32_t)i;
    qsort_r(b->ordinal, b->n, sizeof(uint32_t), cmp_bucket_order, ix); /* total order: no ties */
    b->mz = malloc(b->n * 8);
    b->words = malloc(b->n * ix->W * 8);
    for (size_t r = 0; r < b->n; ++r) { /* :52-56 */
      b->mz[r] = mz[b->ordinal[r]];
      memcpy(b->words + r * ix->W, words + (size_t)b->ordinal[r] * ix->W, ix->W * 8);
    }
  }
  return ix;
}

void ho_index_free(void* h) {
  lib_index* ix = h;
  if (!ix) return;
  for (size_t b = 0; b < ix->n_buckets; ++b) {
    free(ix->buckets[b].mz);
    free(ix->buckets[b].ordinal);
    free(ix->buckets[b].words);
  }
  free(ix->buckets);
  free(ix->mz);
  free(ix->charge);
  free(ix->is_decoy);
  free(ix->id_blob);
  free(ix->id_off);
  free(ix->words_copy);
  free(ix);
}

long long ho_index_bucket_count(const void* h) { return (long long)((const lib_index*)h)->n_buckets; }
long long ho_index_bucket_info(const void* h, uint32_t which, uint8_t* charge, uint64_t* size) {
  const lib_index* ix = h;
  *charge = ix->buckets[which].charge;
  *size = ix->buckets[which].n;
  return 0;
}
long long ho_index_bucket_export(const void* h, uint32_t which, double* mz, uint32_t* ordinal,
                                 uint64_t* words) {
  const lib_index* ix = h;
  const bucket* b = &ix->buckets[which];
  if (mz) memcpy(mz, b->mz, b->n * 8);
  if (ordinal) memcpy(ordinal, b->ordinal, b->n * 4);
  if (words) memcpy(words, b->words, b->n * ix->W * 8);
  return 0;
}

/* ---- tolerance + candidate selection: include/homs/search.hpp:23-30, src/search.cpp:62-89 --- */

static double window_at(int kind, double value, double q) { /* search.hpp:23-25 */
  return kind == 0 ? value * q * 1e-6 : value;
}
static int accepts(int kind, double value, double q, double r) { /* search.hpp:28-30 */
  return fabs(q - r) <= window_at(kind, value, q);
}

static const bucket* bucket_for(const lib_index* ix, uint8_t charge) {
  for (size_t b = 0; b < ix->n_buckets; ++b)
    if (ix->buckets[b].charge == charge) return &ix->buckets[b];
  return NULL;
}

static const bucket* select_candidates(const lib_index* ix, double q, uint8_t charge, int kind,
                                       double value, size_t* first, size_t* last) {
  *first = *last = 0;
  if (charge == 0) return NULL; /* :65 */
  const bucket* b = bucket_for(ix, charge);
  if (!b) return NULL; /* :66-67 */
  const double* mzs = b->mz;
  const size_t n = b->n;
  const double w = window_at(kind, value, q);
  /* std::lower_bound(q - w): first i with !(mz[i] < v); std::upper_bound(q + w): first i with v < mz[i] */
  size_t lo = 0, len = n;
  const double vlo = q - w, vhi = q + w;
  while (len > 0) {
    const size_t half = len / 2;
    if (mzs[lo + half] < vlo) { lo += half + 1; len -= half + 1; } else len = half;
  }
  size_t hi = 0;
  len = n;
  while (len > 0) {
    const size_t half = len / 2;
    if (vhi < mzs[hi + half]) len = half; else { hi += half + 1; len -= half + 1; }
  }
  while (lo > 0 && accepts(kind, value, q, mzs[lo - 1])) --lo;    /* :79 */
  hi = hi > lo ? hi : lo;                                         /* :80 */
  while (hi < n && accepts(kind, value, q, mzs[hi])) ++hi;        /* :81 */
  while (lo < hi && !accepts(kind, value, q, mzs[lo])) ++lo;      /* :82 */
  while (hi > lo && !accepts(kind, value, q, mzs[hi - 1])) --hi;  /* :83 */
  *first = lo;
  *last = hi;
  return b;
}

long long ho_select_candidates(const void* h, uint64_t nq, const double* q_mz,
                               const uint8_t* q_charge, int tol_kind, double tol_value,
                               uint64_t* out_first, uint64_t* out_last, uint8_t* out_has_bucket) {
  const lib_index* ix = h;
  for (uint64_t i = 0; i < nq; ++i) {
    size_t f, l;
    const bucket* b = select_candidates(ix, q_mz[i], q_charge[i], tol_kind, tol_value, &f, &l);
    out_first[i] = f;
    out_last[i] = l;
    out_has_bucket[i] = b != NULL;
  }
  return 0;
}

/* ---- search: src/search.cpp:93-169 ---------------------------------------------------------- */

static uint32_t row_similarity(const uint64_t* row, const uint64_t* q, size_t W, uint32_t dim) {
  uint32_t diff = 0; /* :93-101 */
  for (size_t w = 0; w < W; ++w) diff += popcount64(row[w] ^ q[w]);
  return dim - diff;
}

/* is candidate (score, abs_diff, ordinal a) strictly better than the incumbent? :133-146 */
static int better_than(const lib_index* ix, uint32_t score, double abs_diff, uint32_t ord,
                       uint32_t best_score, double best_abs_diff, uint32_t best_ord) {
  if (score > best_score) return 1;
  if (score == best_score) {
    if (abs_diff < best_abs_diff) return 1;
    if (abs_diff == best_abs_diff) {
      const int c = id_cmp(ix, ord, best_ord);
      return c < 0 || (c == 0 && ord < best_ord);
    }
  }
  return 0;
}

/* returns 1 on hit */
static int search_one(const lib_index* ix, const uint64_t* qw, double q_mz, uint8_t charge,
                      int kind, double value, uint32_t* out_score, uint32_t* out_ord) {
  size_t first, last;
  const bucket* b = select_candidates(ix, q_mz, charge, kind, value, &first, &last);
  if (!b || first >= last) return 0; /* :112 */
  int have = 0;
  uint32_t best_score = 0, best_ord = 0;
  double best_abs = 0.0;
  for (size_t i = first; i < last; ++i) { /* :124-153 */
    const uint32_t score = row_similarity(b->words + i * ix->W, qw, ix->W, ix->dim);
    const double abs_diff = fabs(q_mz - b->mz[i]);
    if (!have || better_than(ix, score, abs_diff, b->ordinal[i], best_score, best_abs, best_ord)) {
      have = 1;
      best_score = score;
      best_abs = abs_diff;
      best_ord = b->ordinal[i];
    }
  }
  *out_score = best_score;
  *out_ord = best_ord;
  return 1;
}

/* tests/oracles.hpp:60-108: exhaustive scan over the input-order library.  NOTE the test
 * oracle breaks (score, |diff|) ties by id only; equal ids keep the earlier entry. */
static int linear_search(const lib_index* ix, const uint64_t* qw, double q_mz, uint8_t charge,
                         int kind, double value, uint32_t* out_score, uint32_t* out_ord) {
  if (charge == 0) return 0;
  int have = 0;
  uint32_t best_score = 0, best = 0;
  double best_diff = 0.0;
  for (size_t i = 0; i < ix->n; ++i) {
    if (ix->charge[i] != charge) continue;
    const double diff = fabs(q_mz - ix->mz[i]);
    const double window = kind == 0 ? value * q_mz * 1e-6 : value;
    if (!(diff <= window)) continue;
    const uint32_t score =
        (uint32_t)ho_hamming_similarity(ix->dim, qw, ix->words_in + i * ix->W, 1);
    int better = 0;
    if (!have || score > best_score) better = 1;
    else if (score == best_score) {
      if (diff < best_diff) better = 1;
      else if (diff == best_diff) better = id_cmp(ix, best, (uint32_t)i) > 0;
    }
    if (better) {
      have = 1;
      best = (uint32_t)i;
      best_score = score;
      best_diff = diff;
    }
  }
  *out_score = best_score;
  *out_ord = best;
  return have;
}

long long ho_search_batch(const void* h, uint64_t nq, const uint64_t* q_words, const double* q_mz,
                          const uint8_t* q_charge, int tol_kind, double tol_value,
                          unsigned threads, uint64_t batch, int linear, uint8_t* out_has,
                          uint32_t* out_raw_score, uint32_t* out_ordinal, double* out_mass_diff) {
  (void)threads;
  (void)batch; /* search.cpp:171-183: elementwise map, scheduling cannot change results */
  const lib_index* ix = h;
  long long hits = 0;
  for (uint64_t i = 0; i < nq; ++i) {
    uint32_t score = 0, ord = 0;
    const int hit = linear ? linear_search(ix, q_words + i * ix->W, q_mz[i], q_charge[i],
                                           tol_kind, tol_value, &score, &ord)
                           : search_one(ix, q_words + i * ix->W, q_mz[i], q_charge[i], tol_kind,
                                        tol_value, &score, &ord);
    out_has[i] = (uint8_t)hit;
    out_raw_score[i] = hit ? score : 0;
    out_ordinal[i] = hit ? ord : 0xFFFFFFFFu;
    if (out_mass_diff) out_mass_diff[i] = hit ? q_mz[i] - ix->mz[ord] : 0.0; /* :164 */
    hits += hit;
  }
  return hits;
}

/* top-k: sort the whole window on the reference key */
typedef struct {
  uint32_t score, ord;
  double abs_diff;
} cand;
static const lib_index* g_sort_ix;
static int cmp_cand(const void* x, const void* y) {
  const cand *a = x, *b = y;
  if (better_than(g_sort_ix, a->score, a->abs_diff, a->ord, b->score, b->abs_diff, b->ord)) return -1;
  if (better_than(g_sort_ix, b->score, b->abs_diff, b->ord, a->score, a->abs_diff, a->ord)) return 1;
  return 0;
}

long long ho_search_topk(const void* h, uint64_t nq, const uint64_t* q_words, const double* q_mz,
                         const uint8_t* q_charge, int tol_kind, double tol_value, uint32_t k,
                         uint32_t* out_raw_score, uint32_t* out_ordinal) {
  const lib_index* ix = h;
  g_sort_ix = ix;
  cand* buf = NULL;
  size_t cap = 0;
  for (uint64_t i = 0; i < nq; ++i) {
    for (uint32_t j = 0; j < k; ++j) {
      out_raw_score[i * k + j] = 0;
      out_ordinal[i * k + j] = 0xFFFFFFFFu;
    }
    size_t first, last;
    const bucket* b = select_candidates(ix, q_mz[i], q_charge[i], tol_kind, tol_value, &first, &last);
    if (!b || first >= last) continue;
    const size_t m = last - first;
    if (m > cap) {
      cap = m;
      buf = realloc(buf, cap * sizeof(cand));
    }
    for (size_t r = 0; r < m; ++r) {
      buf[r].score = row_similarity(b->words + (first + r) * ix->W, q_words + i * ix->W, ix->W, ix->dim);
      buf[r].abs_diff = fabs(q_mz[i] - b->mz[first + r]);
      buf[r].ord = b->ordinal[first + r];
    }
    qsort(buf, m, sizeof(cand), cmp_cand);
    for (uint32_t j = 0; j < k && j < m; ++j) {
      out_raw_score[i * k + j] = buf[j].score;
      out_ordinal[i * k + j] = buf[j].ord;
    }
  }
  free(buf);
  return 0;
}

/* ---- FDR: src/fdr.cpp:8-50 ------------------------------------------------------------------ */

typedef struct {
  const double* score;
  const uint8_t* decoy;
} fdr_ctx;

static int fdr_before(const fdr_ctx* c, uint64_t a, uint64_t b) { /* :17-23 */
  if (c->score[a] != c->score[b]) return c->score[a] > c->score[b];
  return c->decoy[a] > c->decoy[b];
}

static void stable_merge_sort(uint64_t* v, uint64_t* tmp, size_t n, const fdr_ctx* c) {
  if (n < 2) return;
  const size_t h = n / 2;
  stable_merge_sort(v, tmp, h, c);
  stable_merge_sort(v + h, tmp, n - h, c);
  size_t i = 0, j = h, k = 0;
  while (i < h && j < n) tmp[k++] = fdr_before(c, v[j], v[i]) ? v[j++] : v[i++];
  while (i < h) tmp[k++] = v[i++];
  while (j < n) tmp[k++] = v[j++];
  memcpy(v, tmp, n * sizeof(uint64_t));
}

long long ho_compute_fdr_curve(uint64_t n, const double* score, const uint8_t* is_decoy,
                               uint64_t* out_input_index, double* out_fdr, double* out_q) {
  if (n == 0) return 0;
  uint8_t* dec = malloc(n);
  for (uint64_t i = 0; i < n; ++i) dec[i] = is_decoy[i] != 0;
  fdr_ctx c = {score, dec};
  for (uint64_t i = 0; i < n; ++i) out_input_index[i] = i;
  uint64_t* tmp = malloc(n * sizeof(uint64_t));
  stable_merge_sort(out_input_index, tmp, n, &c);
  free(tmp);
  size_t targets = 0, decoys = 0;
  for (uint64_t i = 0; i < n; ++i) { /* :33-43 */
    if (dec[out_input_index[i]]) ++decoys; else ++targets;
    out_fdr[i] = (double)decoys / (double)(targets > 1 ? targets : 1);
  }
  double running = out_fdr[n - 1]; /* :45-50 suffix minimum */
  for (uint64_t i = n; i-- > 0;) {
    running = running < out_fdr[i] ? running : out_fdr[i];
    out_q[i] = running;
  }
  free(dec);
  return (long long)n;
}

/* ---- cascade: src/search.cpp:188-248 -------------------------------------------------------- */

typedef struct {
  int has;
  uint8_t stage;
  uint32_t score, ord;
  double q;
} accepted_t;

static void run_stage(const lib_index* ix, const uint64_t* q_words, const double* q_mz,
                      const uint8_t* q_charge, const uint64_t* todo, size_t n_todo, int kind,
                      double value, uint8_t stage, double fdr_q, accepted_t* accepted) {
  double* score = malloc((n_todo + 1) * sizeof(double));
  uint8_t* decoy = malloc(n_todo + 1);
  uint32_t* raw = malloc((n_todo + 1) * sizeof(uint32_t));
  uint32_t* ord = malloc((n_todo + 1) * sizeof(uint32_t));
  uint64_t* pool_query = malloc((n_todo + 1) * sizeof(uint64_t));
  size_t np = 0;
  for (size_t t = 0; t < n_todo; ++t) { /* :196-207 */
    const uint64_t qi = todo[t];
    uint32_t s, o;
    if (!search_one(ix, q_words + qi * ix->W, q_mz[qi], q_charge[qi], kind, value, &s, &o)) continue;
    raw[np] = s;
    ord[np] = o;
    score[np] = (double)s / (double)ix->dim; /* :165 */
    decoy[np] = ix->is_decoy[o];
    pool_query[np] = qi;
    ++np;
  }
  uint64_t* order = malloc((np + 1) * sizeof(uint64_t));
  double* fdr = malloc((np + 1) * sizeof(double));
  double* q = malloc((np + 1) * sizeof(double));
  ho_compute_fdr_curve(np, score, decoy, order, fdr, q);
  for (size_t p = 0; p < np; ++p) { /* :209-214 */
    const uint64_t in = order[p];
    if (!decoy[in] && q[p] <= fdr_q) {
      accepted_t* a = &accepted[pool_query[in]];
      a->has = 1;
      a->stage = stage;
      a->score = raw[in];
      a->ord = ord[in];
      a->q = q[p];
    }
  }
  free(score); free(decoy); free(raw); free(ord); free(pool_query); free(order); free(fdr); free(q);
}

long long ho_cascade_search(const void* h, uint64_t nq, const uint64_t* q_words,
                            const double* q_mz, const uint8_t* q_charge, int narrow_kind,
                            double narrow_value, int wide_kind, double wide_value, double fdr_q,
                            unsigned threads, uint64_t batch, uint64_t* out_query,
                            uint32_t* out_ordinal, uint8_t* out_stage, uint32_t* out_raw_score,
                            double* out_q_value) {
  (void)threads;
  (void)batch;
  const lib_index* ix = h;
  if (!(narrow_value > 0.0) || !(wide_value > 0.0)) /* :223-224 Tolerance::validate :13-15 */
    return fail("ConfigError", "tolerance value must be positive");
  accepted_t* acc = calloc(nq + 1, sizeof *acc);
  uint64_t* todo = malloc((nq + 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < nq; ++i) todo[i] = i;
  run_stage(ix, q_words, q_mz, q_charge, todo, nq, narrow_kind, narrow_value, 0, fdr_q, acc);
  size_t nr = 0;
  for (uint64_t i = 0; i < nq; ++i)
    if (!acc[i].has) todo[nr++] = i;
  run_stage(ix, q_words, q_mz, q_charge, todo, nr, wide_kind, wide_value, 1, fdr_q, acc);
  long long n = 0;
  for (uint8_t stage = 0; stage < 2; ++stage) /* :240-247 */
    for (uint64_t i = 0; i < nq; ++i)
      if (acc[i].has && acc[i].stage == stage) {
        out_query[n] = i;
        out_ordinal[n] = acc[i].ord;
        out_stage[n] = stage;
        out_raw_score[n] = acc[i].score;
        out_q_value[n] = acc[i].q;
        ++n;
      }
  free(acc);
  free(todo);
  return n;
}

/* ---- synth: src/synth.cpp ------------------------------------------------------------------- */

typedef struct {
  size_t n;
  uint64_t* offsets;
  double *mz, *inten, *precursor;
  uint8_t *charge, *decoy;
  char (*id)[32];
} spec_set;

typedef struct {
  spec_set lib, qry;
  uint64_t* truth_src;
  uint8_t* truth_mod;
} synth_out;

static const double kGridStep = 0.01; /* :25 */

static void make_grid(double mz_min, double mz_max, int64_t* lo_out, int64_t* hi_out) { /* :35-42 */
  int64_t lo = (int64_t)ceil(mz_min / kGridStep - 1e-6);
  int64_t hi = (int64_t)floor(mz_max / kGridStep + 1e-6);
  while (hi >= lo && (double)hi * kGridStep >= mz_max) --hi;
  while (lo <= hi && (double)lo * kGridStep < mz_min) ++lo;
  *lo_out = lo;
  *hi_out = hi;
}

static void random_peptide_draws(mt64* rng, char* out, size_t* len_out) { /* :50-56 */
  static const char kResidues[] = "ACDEFGHIKLMNPQRSTVWY";
  const size_t len = 7 + bounded_uniform(rng, 6);
  for (size_t i = 0; i < len; ++i) out[i] = kResidues[bounded_uniform(rng, 20)];
  *len_out = len;
}

/* :58-77: `count` distinct grid positions, intensities 0.05 + 0.95 u, sorted by m/z */
static void random_peaks(int64_t glo, int64_t ghi, uint32_t count, mt64* rng, uint8_t* used,
                         peak* out) {
  const uint64_t gcount = (uint64_t)(ghi - glo + 1);
  uint32_t m = 0;
  int64_t* picked = malloc(count * sizeof(int64_t));
  while (m < count) {
    const int64_t idx = glo + (int64_t)bounded_uniform(rng, gcount);
    if (used[idx - glo]) continue;
    used[idx - glo] = 1;
    picked[m] = idx;
    out[m].mz = (double)idx * kGridStep;
    out[m].intensity = 0.05 + 0.95 * uniform_unit(rng);
    ++m;
  }
  for (uint32_t i = 0; i < count; ++i) used[picked[i] - glo] = 0;
  free(picked);
  qsort(out, count, sizeof(peak), cmp_mz_asc);
}

static void spec_set_alloc(spec_set* s, size_t n, size_t peaks_cap) {
  s->n = n;
  s->offsets = calloc(n + 1, 8);
  s->mz = malloc((peaks_cap + 1) * 8);
  s->inten = malloc((peaks_cap + 1) * 8);
  s->precursor = calloc(n + 1, 8);
  s->charge = calloc(n + 1, 1);
  s->decoy = calloc(n + 1, 1);
  s->id = calloc(n + 1, 32);
}
static void spec_set_free(spec_set* s) {
  free(s->offsets); free(s->mz); free(s->inten); free(s->precursor);
  free(s->charge); free(s->decoy); free(s->id);
}

void* ho_synth_create(const ho_synthcfg* c) {
  /* SynthConfig::validate :93-112 */
  if (c->n_library < 1) { fail("ConfigError", "synth: n_library must be at least 1"); return NULL; }
  if (c->peaks_per_spectrum < 1) { fail("ConfigError", "synth: need at least one peak"); return NULL; }
  if (!(c->mz_min > 0.0) || !(c->mz_min < c->mz_max)) { fail("ConfigError", "synth: require 0 < mz_min < mz_max"); return NULL; }
  int64_t glo, ghi;
  make_grid(c->mz_min, c->mz_max, &glo, &ghi);
  if (ghi - glo + 1 < (int64_t)c->peaks_per_spectrum) { fail("ConfigError", "synth: peaks_per_spectrum exceeds grid"); return NULL; }
  if (!(c->fraction_modified >= 0.0 && c->fraction_modified <= 1.0) ||
      !(c->fraction_peaks_shifted >= 0.0 && c->fraction_peaks_shifted <= 1.0)) { fail("ConfigError", "synth: fractions must lie in [0, 1]"); return NULL; }
  if (!(c->intensity_noise >= 0.0 && c->intensity_noise < 1.0)) { fail("ConfigError", "synth: intensity_noise must lie in [0, 1)"); return NULL; }
  if (!(c->decoy_ratio >= 0.0)) { fail("ConfigError", "synth: decoy_ratio must be >= 0"); return NULL; }

  const uint32_t P = c->peaks_per_spectrum;
  const double span = c->mz_max - c->mz_min; /* :117-119 */
  const double precursor_lo = c->mz_min + 0.2 * span;
  const double precursor_hi = c->mz_max - 0.2 * span;
  const size_t n_decoys = (size_t)llround(c->decoy_ratio * (double)c->n_library); /* :139-141 */
  const size_t n_lib = c->n_library + n_decoys;

  synth_out* out = calloc(1, sizeof *out);
  spec_set_alloc(&out->lib, n_lib, n_lib * P);
  spec_set_alloc(&out->qry, c->n_query, c->n_query * P);
  out->truth_src = calloc(c->n_query + 1, 8);
  out->truth_mod = calloc(c->n_query + 1, 1);
  uint8_t* used = calloc((size_t)(ghi - glo + 1), 1);
  peak* tmp = malloc(P * sizeof(peak));
  char pep[16];
  size_t pep_len;

  mt64 rng;
  mt64_seed(&rng, stream_seed(c->seed, 0x6c696272617279ULL)); /* "library" :21, :123-134 */
  for (size_t i = 0; i < c->n_library; ++i) {
    snprintf(out->lib.id[i], 32, "LIB_%06zu", i + 1);
    random_peptide_draws(&rng, pep, &pep_len);
    out->lib.charge[i] = (uint8_t)(2 + bounded_uniform(&rng, 2));
    out->lib.precursor[i] = precursor_lo + (precursor_hi - precursor_lo) * uniform_unit(&rng);
    random_peaks(glo, ghi, P, &rng, used, tmp);
    out->lib.offsets[i] = i * P;
    for (uint32_t k = 0; k < P; ++k) {
      out->lib.mz[i * P + k] = tmp[k].mz;
      out->lib.inten[i * P + k] = tmp[k].intensity;
    }
  }
  mt64_seed(&rng, stream_seed(c->seed, 0x6465636f7973ULL)); /* "decoys" :22, :139-157 */
  for (size_t j = 0; j < n_decoys; ++j) {
    const size_t src = j % c->n_library, i = c->n_library + j;
    snprintf(out->lib.id[i], 32, "DECOY_%06zu", j + 1);
    out->lib.charge[i] = out->lib.charge[src];
    out->lib.precursor[i] = out->lib.precursor[src];
    out->lib.decoy[i] = 1;
    random_peaks(glo, ghi, P, &rng, used, tmp);
    out->lib.offsets[i] = i * P;
    for (uint32_t k = 0; k < P; ++k) {
      out->lib.mz[i * P + k] = tmp[k].mz;
      out->lib.inten[i * P + k] = out->lib.inten[src * P + k]; /* :153-155 */
    }
  }
  out->lib.offsets[n_lib] = n_lib * P;

  mt64_seed(&rng, stream_seed(c->seed, 0x71756572696573ULL)); /* "queries" :23, :159-197 */
  uint64_t qp = 0;
  for (size_t q = 0; q < c->n_query; ++q) {
    const size_t src = (size_t)bounded_uniform(&rng, c->n_library);
    snprintf(out->qry.id[q], 32, "QRY_%06zu", q + 1);
    out->qry.charge[q] = out->lib.charge[src];
    double prec = out->lib.precursor[src];
    for (uint32_t k = 0; k < P; ++k) {
      tmp[k].mz = out->lib.mz[src * P + k];
      tmp[k].intensity = out->lib.inten[src * P + k];
    }
    out->truth_src[q] = src;
    const int modified = uniform_unit(&rng) < c->fraction_modified;
    out->truth_mod[q] = (uint8_t)modified;
    if (modified) { /* :176-185 */
      prec += c->precursor_shift_da / (double)out->qry.charge[q];
      for (uint32_t k = 0; k < P; ++k)
        if (uniform_unit(&rng) < c->fraction_peaks_shifted) tmp[k].mz += c->precursor_shift_da;
    }
    if (c->intensity_noise > 0.0) /* :186-191 */
      for (uint32_t k = 0; k < P; ++k) {
        const double u = 2.0 * uniform_unit(&rng) - 1.0;
        tmp[k].intensity *= 1.0 + c->intensity_noise * u;
      }
    qsort(tmp, P, sizeof(peak), cmp_mz_asc); /* sort_and_merge :79-93 */
    out->qry.precursor[q] = prec;
    out->qry.offsets[q] = qp;
    uint64_t start = qp;
    for (uint32_t k = 0; k < P; ++k) {
      if (qp > start && out->qry.mz[qp - 1] == tmp[k].mz) {
        out->qry.inten[qp - 1] += tmp[k].intensity;
      } else {
        out->qry.mz[qp] = tmp[k].mz;
        out->qry.inten[qp] = tmp[k].intensity;
        ++qp;
      }
    }
  }
  out->qry.offsets[c->n_query] = qp;
  free(used);
  free(tmp);
  return out;
}

void ho_synth_free(void* h) {
  synth_out* s = h;
  if (!s) return;
  spec_set_free(&s->lib);
  spec_set_free(&s->qry);
  free(s->truth_src);
  free(s->truth_mod);
  free(s);
}

static const spec_set* pick(const void* h, int which) {
  const synth_out* s = h;
  return which == 0 ? &s->lib : &s->qry;
}

void ho_synth_sizes(const void* h, int which, uint64_t* sizes) {
  const spec_set* s = pick(h, which);
  sizes[0] = s->n;
  sizes[1] = s->offsets[s->n];
  sizes[2] = 0;
  for (size_t i = 0; i < s->n; ++i) sizes[2] += strlen(s->id[i]);
}

void ho_synth_export(const void* h, int which, uint64_t* offsets, double* mz, double* inten,
                     double* precursor, uint8_t* charge, uint8_t* is_decoy, char* id_blob,
                     uint64_t* id_off) {
  const spec_set* s = pick(h, which);
  memcpy(offsets, s->offsets, (s->n + 1) * 8);
  memcpy(mz, s->mz, s->offsets[s->n] * 8);
  memcpy(inten, s->inten, s->offsets[s->n] * 8);
  memcpy(precursor, s->precursor, s->n * 8);
  memcpy(charge, s->charge, s->n);
  memcpy(is_decoy, s->decoy, s->n);
  uint64_t c = 0;
  for (size_t i = 0; i < s->n; ++i) {
    id_off[i] = c;
    const size_t l = strlen(s->id[i]);
    memcpy(id_blob + c, s->id[i], l);
    c += l;
  }
  id_off[s->n] = c;
}

void ho_synth_truth(const void* h, uint64_t* source_index, uint8_t* modified) {
  const synth_out* s = h;
  memcpy(source_index, s->truth_src, s->qry.n * 8);
  memcpy(modified, s->truth_mod, s->qry.n);
}

/* ---- encoded-library cache: src/cache.cpp ------------------------------------------------- */

/* little-endian writers into a growing cursor (cache.cpp:31-57); out may be NULL (sizing pass) */
typedef struct {
  unsigned char* p;
  uint64_t cap, at;
  int overflow;
} wcur;

static void w_bytes(wcur* c, const void* d, uint64_t n) {
  if (c->p) {
    if (c->at + n > c->cap) c->overflow = 1;
    else memcpy(c->p + c->at, d, n);
  }
  c->at += n;
}
static void w_u8(wcur* c, uint8_t v) { w_bytes(c, &v, 1); }
static void w_u32(wcur* c, uint32_t v) {
  unsigned char b[4];
  for (int i = 0; i < 4; ++i) b[i] = (unsigned char)(v >> (8 * i));
  w_bytes(c, b, 4);
}
static void w_u64(wcur* c, uint64_t v) {
  unsigned char b[8];
  for (int i = 0; i < 8; ++i) b[i] = (unsigned char)(v >> (8 * i));
  w_bytes(c, b, 8);
}
static void w_f64(wcur* c, double v) {
  uint64_t u;
  memcpy(&u, &v, 8);
  w_u64(c, u);
}
static void w_str(wcur* c, const char* blob, const uint64_t* off, uint64_t i) { /* cache.cpp:54-57 */
  const uint64_t n = blob && off ? off[i + 1] - off[i] : 0;
  w_u32(c, (uint32_t)n);
  if (n) w_bytes(c, blob + off[i], n);
}
/* put_profile, cache.cpp:98-110: 61 bytes */
static void w_profile(wcur* c, const ho_precfg* pre, const ho_enccfg* enc) {
  w_f64(c, pre->min_mz);
  w_f64(c, pre->max_mz);
  w_f64(c, pre->bin_size);
  w_u32(c, pre->max_peaks);
  w_u32(c, pre->min_peaks);
  w_f64(c, pre->intensity_floor);
  w_u8(c, (uint8_t)pre->scaling);
  w_u32(c, enc->dim);
  w_u32(c, enc->step_flips);
  w_u32(c, enc->levels);
  w_u64(c, enc->seed);
}

long long ho_cache_write(const ho_precfg* pre, const ho_enccfg* enc, uint64_t n, const uint64_t* words,
                         const double* mz, const uint8_t* charge, const uint8_t* is_decoy,
                         const char* id_blob, const uint64_t* id_off, const char* pep_blob,
                         const uint64_t* pep_off, unsigned char* out, uint64_t out_cap) {
  /* write_cache, cache.cpp:122-156 */
  wcur c = {out, out_cap, 0, 0};
  const uint64_t W = ((uint64_t)enc->dim + 63) / 64;
  w_bytes(&c, "HOMS", 4);
  w_u32(&c, 1);
  w_profile(&c, pre, enc);
  w_u64(&c, n);
  for (uint64_t i = 0; i < n; ++i) {
    w_str(&c, id_blob, id_off, i);
    w_f64(&c, mz[i]);
    w_u8(&c, charge[i]);
    w_u8(&c, is_decoy[i] ? 1 : 0);
    w_str(&c, pep_blob, pep_off, i);
  }
  const uint64_t block = c.at;
  for (uint64_t i = 0; i < n * W; ++i) w_u64(&c, words[i]);
  uint64_t digest = 1469598103934665603ULL; /* of the little-endian block bytes */
  if (out && !c.overflow) digest = ho_fnv1a64(out + block, n * W * 8);
  w_u64(&c, digest);
  if (c.overflow) return fail("Error", "ho_cache_write: buffer too small");
  return (long long)c.at;
}

typedef struct {
  const unsigned char* p;
  uint64_t n, at;
  int truncated;
} rcur;

static int r_bytes(rcur* c, void* d, uint64_t n) { /* get_bytes, cache.cpp:59-64 */
  if (c->truncated || c->at + n > c->n) {
    c->truncated = 1;
    memset(d, 0, n);
    return 0;
  }
  memcpy(d, c->p + c->at, n);
  c->at += n;
  return 1;
}
static uint32_t r_u32(rcur* c) {
  unsigned char b[4];
  r_bytes(c, b, 4);
  uint32_t v = 0;
  for (int i = 0; i < 4; ++i) v |= (uint32_t)b[i] << (8 * i);
  return v;
}
static uint64_t r_u64(rcur* c) {
  unsigned char b[8];
  r_bytes(c, b, 8);
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= (uint64_t)b[i] << (8 * i);
  return v;
}

long long ho_cache_read(const unsigned char* image, uint64_t n_bytes, const ho_precfg* pre,
                        const ho_enccfg* enc, uint64_t* words, double* mz, uint8_t* charge,
                        uint8_t* is_decoy, char* id_blob, uint64_t* id_off, char* pep_blob,
                        uint64_t* pep_off) {
  /* read_cache, cache.cpp:158-211; error classes in the reference's order of checks */
  rcur c = {image, n_bytes, 0, 0};
  char magic[4];
  if (!r_bytes(&c, magic, 4)) return fail("CacheCorruptError", "cache stream truncated");
  if (memcmp(magic, "HOMS", 4) != 0) return fail("CacheFormatError", "not a spectral library cache (bad magic)");
  const uint32_t version = r_u32(&c);
  if (c.truncated) return fail("CacheCorruptError", "cache stream truncated");
  if (version != 1) return fail("CacheFormatError", "unsupported cache version");
  unsigned char stored[61], want[61];
  if (!r_bytes(&c, stored, 61)) return fail("CacheCorruptError", "cache stream truncated");
  wcur w = {want, 61, 0, 0};
  w_profile(&w, pre, enc);
  if (memcmp(stored, want, 61) != 0)
    return fail("StaleCacheError", "cache was encoded with different parameters than this run requests");
  const uint64_t count = r_u64(&c);
  if (c.truncated) return fail("CacheCorruptError", "cache stream truncated");
  /* std::vector<EncodedSpectrum> entries(count) would throw bad_alloc on absurd counts; an image
   * cannot hold more entries than it has bytes for their fixed fields */
  if (count > n_bytes / 18) return fail("CacheCorruptError", "cache stream truncated");
  const uint64_t W = ((uint64_t)enc->dim + 63) / 64;
  uint64_t io = 0, po = 0;
  for (uint64_t i = 0; i < count; ++i) {
    for (int which = 0; which < 2; ++which) {
      if (which == 1) { /* between the strings: precursor f64, charge u8, decoy u8 */
        const uint64_t u = r_u64(&c);
        unsigned char cd[2];
        r_bytes(&c, cd, 2);
        if (c.truncated) return fail("CacheCorruptError", "cache stream truncated");
        if (words) {
          memcpy(&mz[i], &u, 8);
          charge[i] = cd[0];
          is_decoy[i] = cd[1] != 0;
        }
      }
      const uint32_t len = r_u32(&c);
      if (c.truncated) return fail("CacheCorruptError", "cache stream truncated");
      if (len > (1u << 20)) return fail("CacheCorruptError", "cache string length out of range");
      if (c.at + len > c.n) return fail("CacheCorruptError", "cache stream truncated");
      if (words) {
        char* blob = which == 0 ? id_blob : pep_blob;
        uint64_t* off = which == 0 ? id_off : pep_off;
        uint64_t* cur = which == 0 ? &io : &po;
        off[i] = *cur;
        memcpy(blob + *cur, c.p + c.at, len);
        *cur += len;
      }
      c.at += len;
    }
  }
  if (words) {
    id_off[count] = io;
    pep_off[count] = po;
  }
  const uint64_t block = count * W * 8;
  if (c.at + block > c.n) return fail("CacheCorruptError", "cache stream truncated");
  const uint64_t digest = ho_fnv1a64(c.p + c.at, block);
  if (words)
    for (uint64_t i = 0; i < count * W; ++i) {
      uint64_t v = 0;
      for (int b = 0; b < 8; ++b) v |= (uint64_t)c.p[c.at + i * 8 + b] << (8 * b);
      words[i] = v;
    }
  c.at += block;
  const uint64_t stored_digest = r_u64(&c);
  if (c.truncated) return fail("CacheCorruptError", "cache stream truncated");
  if (stored_digest != digest) return fail("CacheCorruptError", "cache hypervector block failed its checksum");
  return (long long)count;
}

/* ---- MGF text: src/mgf.cpp ---------------------------------------------------------------------- */

static int mg_space(unsigned char c) {  /* std::isspace in the "C" locale (mgf.cpp:18-26) */
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}
static int mg_alpha(unsigned char c) { return (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z'); }
static int mg_digit(unsigned char c) { return c >= '0' && c <= '9'; }
static int mg_lower(unsigned char c) { return (c >= 'A' && c <= 'Z') ? c + 32 : c; }

static void mg_strip(const char** p, size_t* n) {
  while (*n && mg_space((unsigned char)(*p)[0])) ++*p, --*n;
  while (*n && mg_space((unsigned char)(*p)[*n - 1])) --*n;
}
static size_t mg_first_token(const char* p, size_t n) {  /* mgf.cpp:50-54 */
  size_t i = 0;
  while (i < n && !mg_space((unsigned char)p[i])) ++i;
  return i;
}
static int mg_ieq(const char* p, size_t n, const char* lit) {
  size_t m = strlen(lit);
  if (n != m) return 0;
  for (size_t i = 0; i < n; ++i)
    if (mg_lower((unsigned char)p[i]) != lit[i]) return 0;
  return 1;
}

/* std::from_chars(first, last, double) in chars_format::general that must consume the whole token
 * (mgf.cpp:28-33): optional '-', then inf / infinity / nan / nan(n-char-seq), or digits with an
 * optional '.', and an exponent only when it has digits.  No '+', no hex, no leading blanks.
 * Out-of-range (overflow, or a nonzero value that rounds to zero) is an error. */
static int mg_parse_double(const char* p, size_t n, double* out) {
  size_t i = 0;
  int neg = 0;
  if (i < n && p[i] == '-') neg = 1, ++i;
  if (i < n && mg_alpha((unsigned char)p[i])) {
    if (mg_ieq(p + i, n - i, "inf") || mg_ieq(p + i, n - i, "infinity")) {
      *out = neg ? -INFINITY : INFINITY;
      return 1;
    }
    if (n - i >= 3 && mg_ieq(p + i, 3, "nan")) {
      size_t j = i + 3;
      if (j < n) {
        if (p[j] != '(' || p[n - 1] != ')') return 0;
        for (size_t k = j + 1; k + 1 < n; ++k) {
          unsigned char c = (unsigned char)p[k];
          if (!(mg_alpha(c) || mg_digit(c) || c == '_')) return 0;
        }
      }
      *out = NAN;
      return 1;
    }
    return 0;
  }
  size_t digits = 0;
  int nonzero = 0;
  while (i < n && mg_digit((unsigned char)p[i])) nonzero |= p[i] != '0', ++i, ++digits;
  if (i < n && p[i] == '.') {
    ++i;
    while (i < n && mg_digit((unsigned char)p[i])) nonzero |= p[i] != '0', ++i, ++digits;
  }
  if (digits == 0) return 0;
  if (i < n && (p[i] == 'e' || p[i] == 'E')) {
    size_t j = i + 1;
    if (j < n && (p[j] == '+' || p[j] == '-')) ++j;
    if (j < n && mg_digit((unsigned char)p[j])) {
      while (j < n && mg_digit((unsigned char)p[j])) ++j;
      i = j;
    }
  }
  if (i != n) return 0;
  char stack[128];
  char* buf = n < sizeof stack ? stack : (char*)malloc(n + 1);
  memcpy(buf, p, n);
  buf[n] = 0;
  const double v = strtod(buf, NULL);  /* glibc: correctly rounded, like from_chars */
  if (buf != stack) free(buf);
  if (isinf(v)) return 0;             /* result_out_of_range */
  if (v == 0.0 && nonzero) return 0;  /* underflow to zero: result_out_of_range */
  *out = v;
  return 1;
}

static int mg_parse_charge(const char* p, size_t n, uint8_t* out) {  /* mgf.cpp:35-48 */
  if (n == 0) return 0;
  if (p[0] == '+') ++p, --n;
  else if (p[n - 1] == '+') --n;
  if (n == 0) return 0;
  unsigned long long v = 0;
  for (size_t i = 0; i < n; ++i) {
    if (!mg_digit((unsigned char)p[i])) return 0;
    v = v * 10 + (unsigned)(p[i] - '0');
    if (v > 0xFFFFFFFFull) return 0;  /* from_chars<unsigned>: result_out_of_range */
  }
  if (v < 1 || v > 99) return 0;
  *out = (uint8_t)v;
  return 1;
}

typedef struct {
  double mz, inten;
  size_t seq;
} mg_peak;
static int mg_peak_cmp(const void* a, const void* b) {  /* std::stable_sort by m/z (mgf.cpp:78-79) */
  const mg_peak *x = (const mg_peak*)a, *y = (const mg_peak*)b;
  if (x->mz < y->mz) return -1;
  if (y->mz < x->mz) return 1;
  return x->seq < y->seq ? -1 : (x->seq > y->seq ? 1 : 0);
}

typedef struct {
  uint64_t n, n_peaks, cap, peak_cap, id_bytes, pep_bytes;
  uint64_t* offsets;
  double *mz, *inten, *precursor;
  uint8_t *charge, *decoy;
  char **ids, **peps;
} mg_set;

void ho_mgf_free(void* h) {
  mg_set* s = (mg_set*)h;
  if (!s) return;
  for (uint64_t i = 0; i < s->n; ++i) free(s->ids[i]), free(s->peps[i]);
  free(s->offsets), free(s->mz), free(s->inten), free(s->precursor), free(s->charge), free(s->decoy);
  free(s->ids), free(s->peps), free(s);
}

static void* mg_fail(mg_set* s, mg_peak* pk, size_t line, const char* msg) {
  char buf[200];
  snprintf(buf, sizeof buf, "line %zu: %s", line, msg);  /* errors.hpp:25-27 */
  fail("ParseError", buf);
  free(pk);
  ho_mgf_free(s);
  return NULL;
}

static char* mg_dup(const char* p, size_t n) {
  char* d = (char*)malloc(n + 1);
  memcpy(d, p, n);
  d[n] = 0;
  return d;
}

void* ho_mgf_parse(const char* text, uint64_t n_bytes, const char* decoy_prefix) {
  mg_set* s = (mg_set*)calloc(1, sizeof *s);
  s->offsets = (uint64_t*)calloc(1, sizeof(uint64_t));
  const size_t plen = decoy_prefix ? strlen(decoy_prefix) : 0;
  mg_peak* pk = NULL;
  size_t npk = 0, pk_cap = 0;
  size_t line_no = 0, begin_line = 0, ordinal = 0;
  int inside = 0, has_pepmass = 0;
  double pepmass = 0.0;
  uint8_t charge = 0;
  const char *title = NULL, *pep = NULL;
  size_t title_n = 0, pep_n = 0;

  for (uint64_t pos = 0; pos < n_bytes;) {  /* std::getline, mgf.cpp:100 */
    const char* raw = text + pos;
    const char* nl = (const char*)memchr(raw, '\n', n_bytes - pos);
    size_t len = nl ? (size_t)(nl - raw) : (size_t)(n_bytes - pos);
    pos += len + (nl ? 1 : 0);
    ++line_no;
    const char* line = raw;
    mg_strip(&line, &len);

    if (!inside) {  /* mgf.cpp:104-119 */
      if (len == 0 || line[0] == '#') continue;
      if (len == 10 && memcmp(line, "BEGIN IONS", 10) == 0) {
        inside = 1;
        begin_line = line_no;
        ordinal = s->n + 1;
        has_pepmass = 0, pepmass = 0.0, charge = 0, title = pep = NULL, title_n = pep_n = 0, npk = 0;
        continue;
      }
      if (memchr(line, '=', len) && mg_alpha((unsigned char)line[0])) continue;
      return mg_fail(s, pk, line_no, "unexpected content outside BEGIN IONS/END IONS");
    }
    if (len == 0) continue;
    if (len == 8 && memcmp(line, "END IONS", 8) == 0) {  /* mgf.cpp:122-129, finalize_block :66-89 */
      if (!has_pepmass) return mg_fail(s, pk, begin_line, "spectrum block is missing PEPMASS");
      if (s->n == s->cap) {
        s->cap = s->cap ? 2 * s->cap : 64;
        s->offsets = (uint64_t*)realloc(s->offsets, (s->cap + 1) * sizeof(uint64_t));
        s->precursor = (double*)realloc(s->precursor, s->cap * sizeof(double));
        s->charge = (uint8_t*)realloc(s->charge, s->cap);
        s->decoy = (uint8_t*)realloc(s->decoy, s->cap);
        s->ids = (char**)realloc(s->ids, s->cap * sizeof(char*));
        s->peps = (char**)realloc(s->peps, s->cap * sizeof(char*));
      }
      char idbuf[40];
      const char* id = title;
      size_t id_n = title_n;
      if (title_n == 0) {
        id_n = (size_t)snprintf(idbuf, sizeof idbuf, "spectrum_%zu", ordinal);
        id = idbuf;
      }
      const uint64_t k = s->n;
      s->ids[k] = mg_dup(id, id_n);
      s->peps[k] = mg_dup(pep ? pep : "", pep_n);
      s->id_bytes += id_n;
      s->pep_bytes += pep_n;
      s->precursor[k] = pepmass;
      s->charge[k] = charge;
      s->decoy[k] = plen > 0 && ((id_n >= plen && memcmp(id, decoy_prefix, plen) == 0) ||
                                 (pep_n >= plen && memcmp(pep, decoy_prefix, plen) == 0));
      for (size_t i = 0; i < npk; ++i) pk[i].seq = i;
      qsort(pk, npk, sizeof *pk, mg_peak_cmp);
      if (s->n_peaks + npk > s->peak_cap) {
        s->peak_cap = 2 * (s->n_peaks + npk) + 64;
        s->mz = (double*)realloc(s->mz, s->peak_cap * sizeof(double));
        s->inten = (double*)realloc(s->inten, s->peak_cap * sizeof(double));
      }
      uint64_t w = s->n_peaks;
      for (size_t i = 0; i < npk; ++i) {
        if (w > s->n_peaks && s->mz[w - 1] == pk[i].mz) {
          s->inten[w - 1] += pk[i].inten;  /* duplicate m/z: merge */
        } else {
          s->mz[w] = pk[i].mz;
          s->inten[w] = pk[i].inten;
          ++w;
        }
      }
      s->n_peaks = w;
      s->offsets[k + 1] = w;
      s->n = k + 1;
      inside = 0;
      continue;
    }
    if (len == 10 && memcmp(line, "BEGIN IONS", 10) == 0)
      return mg_fail(s, pk, line_no, "BEGIN IONS inside an open spectrum block");

    if (mg_alpha((unsigned char)line[0])) {  /* mgf.cpp:134-161 */
      const char* eq = (const char*)memchr(line, '=', len);
      if (!eq) return mg_fail(s, pk, line_no, "expected KEY=VALUE header or peak line");
      const size_t key_n = (size_t)(eq - line);
      const char* val = eq + 1;
      size_t val_n = len - key_n - 1;
      mg_strip(&val, &val_n);
      if (key_n == 7 && memcmp(line, "PEPMASS", 7) == 0) {
        double mass = 0.0;
        if (!mg_parse_double(val, mg_first_token(val, val_n), &mass) || !(mass > 0.0))
          return mg_fail(s, pk, line_no, "PEPMASS must be a positive number");
        pepmass = mass;
        has_pepmass = 1;
      } else if (key_n == 6 && memcmp(line, "CHARGE", 6) == 0) {
        if (!mg_parse_charge(val, val_n, &charge))
          return mg_fail(s, pk, line_no, "CHARGE must be a positive integer like 2+");
      } else if (key_n == 5 && memcmp(line, "TITLE", 5) == 0) {
        title = val, title_n = val_n;
      } else if (key_n == 3 && memcmp(line, "SEQ", 3) == 0) {
        pep = val, pep_n = val_n;
      }
      continue;
    }

    /* peak line "mz intensity", extra columns ignored (mgf.cpp:163-177) */
    const size_t mz_n = mg_first_token(line, len);
    const char* rest = line + mz_n;
    size_t rest_n = len - mz_n;
    mg_strip(&rest, &rest_n);
    const size_t in_n = mg_first_token(rest, rest_n);
    double m = 0.0, v = 0.0;
    if (!mg_parse_double(line, mz_n, &m) || !mg_parse_double(rest, in_n, &v))
      return mg_fail(s, pk, line_no, "peak line must be two numbers: m/z intensity");
    if (!(m > 0.0)) return mg_fail(s, pk, line_no, "peak m/z must be positive");
    if (!(v >= 0.0)) return mg_fail(s, pk, line_no, "peak intensity must be non-negative");
    if (npk == pk_cap) {
      pk_cap = pk_cap ? 2 * pk_cap : 256;
      pk = (mg_peak*)realloc(pk, pk_cap * sizeof *pk);
    }
    pk[npk].mz = m;
    pk[npk].inten = v;
    ++npk;
  }
  if (inside) return mg_fail(s, pk, begin_line, "spectrum block not closed by END IONS");
  free(pk);
  return s;
}

void ho_mgf_sizes(const void* h, uint64_t* sizes) {
  const mg_set* s = (const mg_set*)h;
  sizes[0] = s->n, sizes[1] = s->n_peaks, sizes[2] = s->id_bytes, sizes[3] = s->pep_bytes;
}

void ho_mgf_export(const void* h, uint64_t* offsets, double* mz, double* inten, double* precursor,
                   uint8_t* charge, uint8_t* is_decoy, char* id_blob, uint64_t* id_off, char* pep_blob,
                   uint64_t* pep_off) {
  const mg_set* s = (const mg_set*)h;
  memcpy(offsets, s->offsets, (s->n + 1) * sizeof(uint64_t));
  if (s->n_peaks) {
    memcpy(mz, s->mz, s->n_peaks * sizeof(double));
    memcpy(inten, s->inten, s->n_peaks * sizeof(double));
  }
  uint64_t c = 0, q = 0;
  for (uint64_t i = 0; i < s->n; ++i) {
    precursor[i] = s->precursor[i];
    charge[i] = s->charge[i];
    is_decoy[i] = s->decoy[i];
    id_off[i] = c;
    pep_off[i] = q;
    const size_t a = strlen(s->ids[i]), b = strlen(s->peps[i]);
    memcpy(id_blob + c, s->ids[i], a);
    memcpy(pep_blob + q, s->peps[i], b);
    c += a;
    q += b;
  }
  id_off[s->n] = c;
  pep_off[s->n] = q;
}

long long ho_mgf_write(uint64_t n, const uint64_t* offsets, const double* mz, const double* inten,
                       const double* precursor, const uint8_t* charge, const char* id_blob,
                       const uint64_t* id_off, const char* pep_blob, const uint64_t* pep_off, char* out,
                       uint64_t cap) {  /* mgf.cpp:183-208 */
  uint64_t w = 0;
  char buf[96];
#define MG_PUT(ptr, len)                                    \
  do {                                                      \
    if (out && w + (len) <= cap) memcpy(out + w, (ptr), (len)); \
    w += (len);                                             \
  } while (0)
  for (uint64_t i = 0; i < n; ++i) {
    MG_PUT("BEGIN IONS\nTITLE=", 17);
    MG_PUT(id_blob + id_off[i], id_off[i + 1] - id_off[i]);
    int k = snprintf(buf, sizeof buf, "\nPEPMASS=%.5f\n", precursor[i]);
    MG_PUT(buf, (uint64_t)k);
    if (charge[i] != 0) {
      k = snprintf(buf, sizeof buf, "CHARGE=%u+\n", (unsigned)charge[i]);
      MG_PUT(buf, (uint64_t)k);
    }
    if (pep_blob && pep_off[i + 1] > pep_off[i]) {
      MG_PUT("SEQ=", 4);
      MG_PUT(pep_blob + pep_off[i], pep_off[i + 1] - pep_off[i]);
      MG_PUT("\n", 1);
    }
    for (uint64_t j = offsets[i]; j < offsets[i + 1]; ++j) {
      k = snprintf(buf, sizeof buf, "%.5f %.6f\n", mz[j], inten[j]);
      MG_PUT(buf, (uint64_t)k);
    }
    MG_PUT("END IONS\n\n", 10);
  }
#undef MG_PUT
  return (long long)w;
}
