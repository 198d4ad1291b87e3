/*
 * miso_oracle.c -- CPU restatement of the MISO decision core. TEST INFRASTRUCTURE ONLY:
 * the checker for the CUDA path, never the measured or shipped path (see miso_oracle.h).
 * Reference paths are relative to /root/reference/proj/include/miso/.
 */
#include "miso_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================== */
/* common.hpp:70-119 -- splitmix64, mix_seed, DetRng over std::mt19937_64    */
/* ======================================================================== */

uint64_t orc_splitmix64(uint64_t x) { /* common.hpp:70-75 */
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

uint64_t orc_mix_seed(uint64_t seed, uint64_t tag) { /* common.hpp:77-79 */
  return orc_splitmix64(orc_splitmix64(seed) ^ orc_splitmix64(tag));
}

/* std::mt19937_64 as pinned by [rand.predef]: w=64 n=312 m=156 r=31. */
void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = 312;
}

uint64_t orc_rng_raw(orc_rng* r) {
  static const uint64_t mag[2] = {0ull, 0xB5026F5AA96619E9ull};
  const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  if (r->mti >= 312) {
    int i;
    for (i = 0; i < 312 - 156; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ mag[x & 1];
    }
    for (; i < 311; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + 156 - 312] ^ (x >> 1) ^ mag[x & 1];
    }
    uint64_t x = (r->mt[311] & UM) | (r->mt[0] & LM);
    r->mt[311] = r->mt[155] ^ (x >> 1) ^ mag[x & 1];
    r->mti = 0;
  }
  uint64_t y = r->mt[r->mti++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

double orc_uniform01(orc_rng* r) { return (double)(orc_rng_raw(r) >> 11) * 0x1.0p-53; }
double orc_uniform(orc_rng* r, double lo, double hi) { return lo + (hi - lo) * orc_uniform01(r); }
double orc_exponential(orc_rng* r, double mean) {
  double u = orc_uniform01(r);
  return -mean * log1p(-u);
}
double orc_normal01(orc_rng* r) { /* common.hpp:103-108 */
  double u1 = orc_uniform01(r);
  double u2 = orc_uniform01(r);
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925287 * u2);
}
double orc_lognormal(orc_rng* r, double mu, double sigma) { return exp(mu + sigma * orc_normal01(r)); }
int orc_index(orc_rng* r, int n) { return (int)(orc_rng_raw(r) % (uint64_t)n); }

/* ======================================================================== */
/* topology.hpp                                                              */
/* ======================================================================== */

const int orc_gpc[ORC_KINDS] = {1, 2, 3, 4, 7};        /* topology.hpp:39-45 */
const int orc_mem_gb[ORC_KINDS] = {5, 10, 20, 20, 40};
const int orc_units[ORC_KINDS] = {1, 2, 4, 4, 8};
const int orc_max_count[ORC_KINDS] = {7, 3, 2, 1, 1};

int orc_violation(const uint8_t c[ORC_KINDS]) { /* topology.hpp:84-101 */
  int total = 0, gpc = 0, mem = 0;
  for (int k = 0; k < ORC_KINDS; ++k) {
    if (c[k] > orc_max_count[k]) return 1;
    total += c[k];
    gpc += c[k] * orc_gpc[k];
    mem += c[k] * orc_units[k];
  }
  if (total == 0) return 2;
  if (gpc > 7) return 3;
  if (mem > 8) return 4;
  if (c[3] > 0 && c[2] > 0) return 5;
  return 0;
}

/* slices_desc -> gpc vector (topology.hpp:137-147) */
static int gpc_vector(const uint8_t c[ORC_KINDS], int v[7]) {
  int n = 0;
  for (int k = ORC_KINDS - 1; k >= 0; --k)
    for (int i = 0; i < c[k]; ++i) v[n++] = orc_gpc[k];
  return n;
}

/* std::vector<int> operator< : lexicographic, shorter prefix first */
static int lex_cmp(const int* a, int na, const int* b, int nb) {
  int n = na < nb ? na : nb;
  for (int i = 0; i < n; ++i)
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  return na == nb ? 0 : (na < nb ? -1 : 1);
}

static int catalog_order_cmp(const void* pa, const void* pb) { /* topology.hpp:178-180 */
  int va[7], vb[7];
  int na = gpc_vector((const uint8_t*)pa, va), nb = gpc_vector((const uint8_t*)pb, vb);
  return -lex_cmp(va, na, vb, nb); /* descending */
}

void orc_build_catalog(orc_catalog* cat) { /* topology.hpp:189-202 */
  uint8_t c[ORC_KINDS];
  cat->n_entries = 0;
  for (c[4] = 0; c[4] <= 1; ++c[4])
    for (c[3] = 0; c[3] <= 1; ++c[3])
      for (c[2] = 0; c[2] <= 2; ++c[2])
        for (c[1] = 0; c[1] <= 3; ++c[1])
          for (c[0] = 0; c[0] <= 7; ++c[0])
            if (!orc_violation(c)) memcpy(cat->counts[cat->n_entries++], c, ORC_KINDS);
  /* std::sort is not stable, but catalog_order is a strict total order on distinct
   * multisets (distinct counts => distinct gpc vectors), so any sort agrees. */
  qsort(cat->counts, (size_t)cat->n_entries, ORC_KINDS, catalog_order_cmp);
}

static int slice_count(const uint8_t c[ORC_KINDS]) {
  int n = 0;
  for (int k = 0; k < ORC_KINDS; ++k) n += c[k];
  return n;
}
static int total_gpc(const uint8_t c[ORC_KINDS]) {
  int g = 0;
  for (int k = 0; k < ORC_KINDS; ++k) g += c[k] * orc_gpc[k];
  return g;
}

/* std::next_permutation on a small int array */
static int next_perm(int* a, int n) {
  int i = n - 2;
  while (i >= 0 && a[i] >= a[i + 1]) --i;
  if (i < 0) {
    for (int l = 0, r = n - 1; l < r; ++l, --r) { int t = a[l]; a[l] = a[r]; a[r] = t; }
    return 0;
  }
  int j = n - 1;
  while (a[j] <= a[i]) --j;
  int t = a[i]; a[i] = a[j]; a[j] = t;
  for (int l = i + 1, r = n - 1; l < r; ++l, --r) { t = a[l]; a[l] = a[r]; a[r] = t; }
  return 1;
}

typedef struct {
  int entry, m, tg;
  int shape[7];
  int place[7];
} cand_tmp;

/* OptKey::beats minus the objective (optimizer.hpp:46-51): total_gpc asc, shape asc,
 * placement asc. A static total order, so a rank-ordered scan with strict '>' on the
 * objective reproduces the reference argmax. */
static int cand_cmp(const void* pa, const void* pb) {
  const cand_tmp* a = (const cand_tmp*)pa;
  const cand_tmp* b = (const cand_tmp*)pb;
  if (a->m != b->m) return a->m < b->m ? -1 : 1;
  if (a->tg != b->tg) return a->tg < b->tg ? -1 : 1;
  int c = lex_cmp(a->shape, a->m, b->shape, b->m);
  if (c) return c;
  return lex_cmp(a->place, a->m, b->place, b->m);
}

void orc_build_candidates(orc_candidates* out) {
  orc_catalog cat;
  orc_build_catalog(&cat);
  cand_tmp tmp[ORC_MAX_CANDS];
  int n = 0;
  for (int e = 0; e < cat.n_entries; ++e) {
    const uint8_t* c = cat.counts[e];
    int m = slice_count(c);
    int perm[7], k = 0;
    for (int kind = 0; kind < ORC_KINDS; ++kind) /* ascending start (optimizer.hpp:75-76) */
      for (int i = 0; i < c[kind]; ++i) perm[k++] = kind;
    do {
      cand_tmp* t = &tmp[n++];
      t->entry = e;
      t->m = m;
      t->tg = total_gpc(c);
      gpc_vector(c, t->shape);
      memcpy(t->place, perm, sizeof(int) * (size_t)m);
    } while (next_perm(perm, m));
  }
  qsort(tmp, (size_t)n, sizeof(cand_tmp), cand_cmp);
  out->n = n;
  for (int m = 0; m <= 8; ++m) out->base[m] = 0;
  for (int i = 0; i < n; ++i) {
    out->entry[i] = (uint8_t)tmp[i].entry;
    out->m[i] = (uint8_t)tmp[i].m;
    memset(out->place[i], 0, 7);
    for (int j = 0; j < tmp[i].m; ++j) out->place[i][j] = (uint8_t)tmp[i].place[j];
  }
  for (int m = 1; m <= 8; ++m) {
    int b = 0;
    while (b < n && out->m[b] < m) ++b;
    out->base[m] = b;
  }
  out->base[0] = 0;
}

int orc_min_slice_for(int mem_gb, int qos_min_gpc) { /* topology.hpp:68-72 */
  for (int k = 0; k < ORC_KINDS; ++k)
    if (orc_mem_gb[k] >= mem_gb && orc_gpc[k] >= qos_min_gpc) return k;
  return -1;
}

int orc_max_spare_slice_for(const orc_catalog* cat, const int* min_kinds_in, int m) {
  /* topology.hpp:227-252 */
  if (m >= 7) return -1;
  int mk[7];
  memcpy(mk, min_kinds_in, sizeof(int) * (size_t)m);
  for (int i = 1; i < m; ++i) /* sort descending */
    for (int j = i; j > 0 && mk[j - 1] < mk[j]; --j) { int t = mk[j]; mk[j] = mk[j - 1]; mk[j - 1] = t; }
  int best = -1;
  for (int e = 0; e < cat->n_entries; ++e) {
    const uint8_t* c = cat->counts[e];
    if (slice_count(c) != m + 1) continue;
    int sl[7], ns = 0;
    for (int k = ORC_KINDS - 1; k >= 0; --k)
      for (int i = 0; i < c[k]; ++i) sl[ns++] = k;
    for (int spare = 0; spare < ns; ++spare) {
      if (spare > 0 && sl[spare] == sl[spare - 1]) continue;
      if (best >= 0 && sl[spare] <= best) continue;
      int ok = 1, j = 0;
      for (int i = 0; i < ns && ok; ++i) {
        if (i == spare) continue;
        if (sl[i] < mk[j]) ok = 0;
        ++j;
      }
      if (ok) best = sl[spare];
    }
  }
  return best;
}

/* Sorted multiset of m <= 6 kinds (values 0..4) -> dense key in [0, 462):
 * key = offset(m) + combinatorial rank of the non-decreasing sequence. */
static int multiset_count(int len, int maxv) { /* # non-decreasing seqs of length len over [0,maxv] */
  /* C(len + maxv, maxv) */
  int num = 1, den = 1;
  for (int i = 1; i <= maxv; ++i) { num *= len + i; den *= i; }
  return num / den;
}

int orc_spare_key(const int* kinds, int m) {
  int s[6];
  memcpy(s, kinds, sizeof(int) * (size_t)m);
  for (int i = 1; i < m; ++i)
    for (int j = i; j > 0 && s[j - 1] > s[j]; --j) { int t = s[j]; s[j] = s[j - 1]; s[j - 1] = t; }
  int key = 0;
  for (int l = 0; l < m; ++l) key += multiset_count(l, 4);
  /* rank of s among non-decreasing sequences of length m over [0,4] */
  int lo = 0;
  for (int i = 0; i < m; ++i) {
    for (int v = lo; v < s[i]; ++v) key += multiset_count(m - i - 1, 4 - v);
    lo = s[i];
  }
  return key;
}

static void spare_lut_rec(const orc_catalog* cat, int8_t* lut, int* s, int pos, int m, int lo) {
  if (pos == m) {
    lut[orc_spare_key(s, m)] = (int8_t)orc_max_spare_slice_for(cat, s, m);
    return;
  }
  for (int v = lo; v < ORC_KINDS; ++v) {
    s[pos] = v;
    spare_lut_rec(cat, lut, s, pos + 1, m, v);
  }
}

void orc_build_spare_lut(const orc_catalog* cat, int8_t lut[462]) {
  int s[6];
  for (int m = 0; m <= 6; ++m) spare_lut_rec(cat, lut, s, 0, m, 0);
}

/* ======================================================================== */
/* optimizer.hpp:62-115 -- literal restatement (next_permutation enumeration) */
/* ======================================================================== */

typedef struct {
  double obj;
  int tg, m;
  int shape[7];
  int place[7];
} opt_key;

static int key_beats(const opt_key* a, const opt_key* b) { /* optimizer.hpp:46-51 */
  if (a->obj != b->obj) return a->obj > b->obj;
  if (a->tg != b->tg) return a->tg < b->tg;
  int c = lex_cmp(a->shape, a->m, b->shape, b->m);
  if (c) return c < 0;
  return lex_cmp(a->place, a->m, b->place, b->m) < 0;
}

int orc_optimize(const orc_catalog* cat, const double* speeds, int m, int* entry, uint8_t* place,
                 double* objective) {
  if (m < 1 || m > 7) return -1; /* optimizer.hpp:65-66 throws invalid_argument */
  opt_key best;
  int found = 0, best_e = -1;
  for (int e = 0; e < cat->n_entries; ++e) {
    const uint8_t* c = cat->counts[e];
    if (slice_count(c) != m) continue;
    int perm[7], k = 0;
    for (int kind = 0; kind < ORC_KINDS; ++kind)
      for (int i = 0; i < c[kind]; ++i) perm[k++] = kind;
    do {
      double obj = 0; /* optimizer.hpp:78-87: FP64 sum in job order */
      int valid = 1;
      for (int i = 0; i < m; ++i) {
        double v = speeds[i * ORC_KINDS + perm[i]];
        if (!(v > 0)) { valid = 0; break; }
        obj += v;
      }
      if (!valid) continue;
      opt_key key;
      key.obj = obj;
      key.tg = total_gpc(c);
      key.m = m;
      gpc_vector(c, key.shape);
      memcpy(key.place, perm, sizeof(int) * (size_t)m);
      if (!found || key_beats(&key, &best)) {
        best = key;
        best_e = e;
        found = 1;
      }
    } while (next_perm(perm, m));
  }
  if (!found) return 0; /* optimizer.hpp:102 nullopt */
  *entry = best_e;
  for (int i = 0; i < m; ++i) place[i] = (uint8_t)best.place[i];
  *objective = best.obj;
  return 1;
}

void orc_optimize_batch(const orc_catalog* cat, const double* speeds, const uint32_t* offsets,
                        size_t n, int16_t* entry, uint8_t* place, double* obj) {
  for (size_t i = 0; i < n; ++i) {
    uint32_t o = offsets[i];
    int m = (int)(offsets[i + 1] - o);
    int e = -1;
    double ob = 0;
    int r = orc_optimize(cat, speeds + (size_t)o * ORC_KINDS, m, &e, place + o, &ob);
    entry[i] = (int16_t)(r == 1 ? e : (r == 0 ? -1 : -2));
    obj[i] = r == 1 ? ob : 0.0;
  }
}

/* ======================================================================== */
/* profiles.hpp                                                              */
/* ======================================================================== */

#define SPEED_FLOOR 1e-9 /* profiles.hpp:33 kSpeedFloor */

static double clampd(double v, double lo, double hi) { /* std::clamp */
  return v < lo ? lo : (hi < v ? hi : v);
}

double orc_effective_speed(double speed, int kind, int mem_gb, int qos_kind) { /* :60-65 */
  if (orc_mem_gb[kind] < mem_gb) return 0.0;
  if (qos_kind >= 0 && orc_gpc[kind] < orc_gpc[qos_kind]) return 0.0;
  return speed;
}

double orc_perturb_speed(double truth, double target_mae, uint64_t entry_seed) { /* :193-205 */
  if (target_mae <= 0.0) return truth;
  orc_rng rng;
  orc_rng_seed(&rng, entry_seed);
  const double sigma = target_mae * sqrt(3.14159265358979323846 / 2.0);
  const double mag = fabs(orc_normal01(&rng)) * sigma;
  const int up_ok = truth + mag <= 1.0;
  const int dn_ok = truth - mag >= SPEED_FLOOR;
  const int coin = orc_uniform01(&rng) < 0.5;
  if (up_ok && dn_ok) return coin ? truth + mag : truth - mag;
  if (up_ok) return truth + mag;
  if (dn_ok) return truth - mag;
  return (1.0 - truth >= truth - SPEED_FLOOR) ? 1.0 : SPEED_FLOOR;
}

void orc_predict_column(const double t[3], int col, uint64_t rng_seed, uint64_t nonce, int noisy,
                        double target_mae, double out[3]) {
  /* profiles.hpp:234-248 for one non-dummy column */
  for (int r = 0; r < 3; ++r) {
    if (!noisy || r == 0) {
      out[r] = t[r];
    } else {
      uint64_t es = orc_mix_seed(orc_mix_seed(rng_seed, nonce), (uint64_t)col * 8 + (uint64_t)r);
      out[r] = orc_perturb_speed(t[r], target_mae, es);
    }
  }
  double mx = out[0]; /* std::max({a,b,c}) keeps the first of equal maxima */
  if (mx < out[1]) mx = out[1];
  if (mx < out[2]) mx = out[2];
  for (int r = 0; r < 3; ++r) out[r] = clampd(out[r] / mx, SPEED_FLOOR, 1.0);
}

void orc_extrapolate(const double w2[4], const double w1[4], const double f[3], double* f2,
                     double* f1) { /* profiles.hpp:267-272, 376-381 */
  double p2 = w2[0] * f[0] + w2[1] * f[1] + w2[2] * f[2] + w2[3];
  double p1 = w1[0] * f[0] + w1[1] * f[1] + w1[2] * f[2] + w1[3];
  *f2 = clampd(p2, SPEED_FLOOR, f[2]);
  *f1 = clampd(p1, SPEED_FLOOR, *f2);
}

void orc_predict_batch(const double* truth3, size_t ncols, int cpg, uint64_t first_nonce,
                       uint64_t rng_seed, int noisy, double target_mae, const double w2[4],
                       const double w1[4], double* out5) {
  for (size_t j = 0; j < ncols; ++j) {
    double f[3], f2, f1;
    orc_predict_column(truth3 + 3 * j, (int)(j % (size_t)cpg), rng_seed,
                       first_nonce + j / (size_t)cpg, noisy, target_mae, f);
    orc_extrapolate(w2, w1, f, &f2, &f1);
    double* o = out5 + 5 * j;
    o[0] = f1; o[1] = f2; o[2] = f[2]; o[3] = f[1]; o[4] = f[0];
  }
}

static double interp_speed(const double v[5], double gpc) { /* profiles.hpp:391-402 */
  static const double knots[5] = {1, 2, 3, 4, 7};
  if (gpc <= knots[0]) return v[0];
  if (gpc >= knots[4]) return v[4];
  for (int i = 1; i < 5; ++i)
    if (gpc <= knots[i]) {
      double w = (gpc - knots[i - 1]) / (knots[i] - knots[i - 1]);
      return v[i - 1] + w * (v[i] - v[i - 1]);
    }
  return v[4];
}

void orc_synthetic_profile(orc_rng* r, double v[5], int* mem_gb, double mps[3]) { /* :443-465 */
  double alpha = orc_uniform(r, 0.1, 1.0);
  for (int k = 0; k < 5; ++k) {
    double base = pow(orc_gpc[k] / 7.0, alpha);
    v[k] = base * (1.0 + orc_uniform(r, -0.03, 0.03));
  }
  double anchor = v[4];
  for (int k = 0; k < 5; ++k) v[k] /= anchor;
  v[4] = 1.0;
  for (int i = 3; i >= 0; --i) v[i] = clampd(v[i], 1e-6, v[i + 1]);
  double u = orc_uniform01(r);
  *mem_gb = u < 4.0 / 9.0 ? 5 : (u < 7.0 / 9.0 ? 10 : 20);
  mps[0] = 1.0;
  mps[1] = clampd(interp_speed(v, 3.5), SPEED_FLOOR, 1.0);
  mps[2] = v[0];
}

/* profiles.hpp:279-332 -- cyclic Jacobi + min-norm pseudo-inverse solve */
static void jacobi_eigen3(double a[3][3], double vals[3], double vecs[3][3]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) vecs[i][j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
    if (off < 1e-300) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (fabs(a[p][q]) < 1e-300) continue;
        double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        double sgn = theta >= 0 ? 1.0 : -1.0;
        double tgt = sgn / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(tgt * tgt + 1.0);
        double s = tgt * c;
        for (int k = 0; k < 3; ++k) {
          double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          double vkp = vecs[k][p], vkq = vecs[k][q];
          vecs[k][p] = c * vkp - s * vkq;
          vecs[k][q] = s * vkp + c * vkq;
        }
      }
  }
  for (int i = 0; i < 3; ++i) vals[i] = a[i][i];
}

static void solve_min_norm(double ata_in[3][3], const double aty[3], double w[3]) {
  double a[3][3], vals[3], vecs[3][3];
  memcpy(a, ata_in, sizeof(a));
  jacobi_eigen3(a, vals, vecs);
  double lmax = fabs(vals[0]);
  if (lmax < fabs(vals[1])) lmax = fabs(vals[1]);
  if (lmax < fabs(vals[2])) lmax = fabs(vals[2]);
  double tol = lmax * 1e-12;
  w[0] = w[1] = w[2] = 0;
  for (int e = 0; e < 3; ++e) {
    if (fabs(vals[e]) <= tol) continue;
    double proj = 0;
    for (int k = 0; k < 3; ++k) proj += vecs[k][e] * aty[k];
    proj /= vals[e];
    for (int k = 0; k < 3; ++k) w[k] += vecs[k][e] * proj;
  }
}

void orc_default_model(double w2o[4], double w1o[4]) {
  /* sim.hpp:894-898: fit_small_slice_model(make_training_corpus(3000, 0x5eed)) */
  orc_rng r;
  orc_rng_seed(&r, orc_mix_seed(0x5eedull, 0x7261696eull)); /* profiles.hpp:469-475 */
  double ata[3][3] = {{0}}, aty2[3] = {0}, aty1[3] = {0};
  for (int n = 0; n < 3000; ++n) {
    double v[5], mps[3];
    int mem;
    orc_synthetic_profile(&r, v, &mem, mps);
    double x[3] = {v[3], v[2], 1.0};
    for (int i = 0; i < 3; ++i) {
      for (int j = 0; j < 3; ++j) ata[i][j] += x[i] * x[j];
      aty2[i] += x[i] * v[1];
      aty1[i] += x[i] * v[0];
    }
  }
  double w2[3], w1[3];
  solve_min_norm(ata, aty2, w2);
  solve_min_norm(ata, aty1, w1);
  w2o[0] = 0.0; w2o[1] = w2[0]; w2o[2] = w2[1]; w2o[3] = w2[2];
  w1o[0] = 0.0; w1o[1] = w1[0]; w1o[2] = w1[1]; w1o[3] = w1[2];
}

/* ======================================================================== */
/* generators                                                                */
/* ======================================================================== */

size_t orc_gen_mixes(uint64_t seed, size_t n, double* speeds, uint32_t* offsets,
                     size_t max_jobs) {
  /* acceptance_test.cpp:72-85 */
  orc_rng r;
  orc_rng_seed(&r, seed);
  size_t jobs = 0;
  offsets[0] = 0;
  for (size_t t = 0; t < n; ++t) {
    int m = 1 + orc_index(&r, 7);
    if (jobs + (size_t)m > max_jobs) return (size_t)-1;
    for (int i = 0; i < m; ++i) {
      double f4 = orc_uniform(&r, 0.2, 1.0);
      double f3 = orc_uniform(&r, 0.15, f4);
      double f2 = orc_uniform(&r, 0.1, f3);
      double f1 = orc_uniform(&r, 0.05, f2);
      if (orc_uniform01(&r) < 0.25) f1 = 0.0;
      double* v = speeds + 5 * (jobs + (size_t)i);
      v[0] = f1; v[1] = f2; v[2] = f3; v[3] = f4; v[4] = 1.0;
    }
    jobs += (size_t)m;
    offsets[t + 1] = (uint32_t)jobs;
  }
  return jobs;
}

void orc_gen_profiles(uint64_t seed, size_t n, double* truth3, double* small2) {
  orc_rng r;
  orc_rng_seed(&r, orc_mix_seed(seed, 0x50));
  for (size_t i = 0; i < n; ++i) {
    double v[5], mps[3];
    int mem;
    orc_synthetic_profile(&r, v, &mem, mps);
    truth3[3 * i + 0] = v[4];
    truth3[3 * i + 1] = v[3];
    truth3[3 * i + 2] = v[2];
    if (small2) { small2[2 * i] = v[1]; small2[2 * i + 1] = v[0]; }
  }
}
