/*
 * gen/pencil_gen.c -- seeded synthetic pencils in generalized real Schur form.
 *
 * Shared input generator for tests, smoke() and bench.py.  It holds none of the
 * method's arithmetic: it only draws random numbers and places them.  The recipe is the
 * one of DESIGN.md section "Inputs" (BASELINE.json configs[0..4]; it stands in for the
 * paper's starneig-test generator, which is not available):
 *
 *   1x1 block: s ~ U[-1,1], t ~ U[0.5,1.5]                         (eigenvalue s/t)
 *   2x2 block: T_blk = diag(t1,t2), t ~ U[0.5,1.5];
 *              S_blk = [[a, b], [-c, a t2/t1]], a ~ U[-1,1], b,c ~ U[0.1,1]
 *              (eigenvalues a/t1 +- i sqrt(bc/(t1 t2)))
 *   strictly-upper entries outside the 2x2 blocks: N(0, var_off) in S and in T;
 *   T_blk(1,2) = 0; all strictly-lower entries 0 except the 2x2 subdiagonals of S.
 *   Block kinds are placed in random order (Fisher-Yates).
 *   Optional: zero / infinite eigenvalues (s = 0 / t = 0 for chosen 1x1 blocks);
 *   eigenvalue separation (whole-pencil reseed, or per-eigenvalue redraw);
 *   overflow stress: a fraction of the strictly-upper tiles of a fixed generator grid
 *   scaled by a factor in S and T, and real eigenvalues in clusters.
 *
 * RNG: Philox4x32-10, key = seed, counter = (index lo, index hi, stream tag, attempt).
 * Each draw gives two 53-bit uniforms.  A normal is sqrt(-2 ln u1) cos(2 pi u2) (host libm).
 * The pencil is bit-identical for any thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { TAG_PERM = 1, TAG_DIAG = 2, TAG_OFFS = 3, TAG_OFFT = 4, TAG_TILES = 5, TAG_CLUS = 6,
       TAG_SPECIAL = 7 };

static void philox(uint32_t c[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
  uint32_t x0 = c[0], x1 = c[1], x2 = c[2], x3 = c[3];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * x0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * x2;
    uint32_t y0 = (uint32_t)(p1 >> 32) ^ x1 ^ k0;
    uint32_t y1 = (uint32_t)p1;
    uint32_t y2 = (uint32_t)(p0 >> 32) ^ x3 ^ k1;
    uint32_t y3 = (uint32_t)p0;
    x0 = y0; x1 = y1; x2 = y2; x3 = y3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

/* two uniforms in [0,1) from one draw keyed by (seed, tag, index, attempt) */
static void uni2(uint64_t seed, uint32_t tag, uint64_t index, uint32_t attempt, double u[2]) {
  uint32_t c[4] = {(uint32_t)index, (uint32_t)(index >> 32), tag, attempt};
  uint32_t o[4];
  philox(c, (uint32_t)seed, (uint32_t)(seed >> 32), o);
  u[0] = (double)(((uint64_t)(o[0] >> 5) << 26) | (o[1] >> 6)) * 0x1p-53;
  u[1] = (double)(((uint64_t)(o[2] >> 5) << 26) | (o[3] >> 6)) * 0x1p-53;
}

static double normal(uint64_t seed, uint32_t tag, uint64_t index) {
  double u[2];
  uni2(seed, tag, index, 0, u);
  return sqrt(-2.0 * log(1.0 - u[0])) * cos(6.283185307179586 * u[1]);
}

typedef struct {
  int m, n2;
  double var_off;        /* variance of the off-diagonal normals */
  uint64_t seed;
  int gap_mode;          /* 0 none, 1 whole-pencil reseed, 2 per-eigenvalue redraw */
  double gap;            /* min |lambda_i - lambda_j| */
  int n_zero, n_inf;     /* 1x1 blocks turned into zero / infinite eigenvalues */
  double stress_frac;    /* fraction of strictly-upper generator tiles scaled */
  int stress_tile;       /* generator tile size (128) */
  double stress_scale;   /* factor (1e100) */
  int cluster;           /* real eigenvalues in clusters of this size (0 = off) */
  double cluster_gap;    /* spacing inside a cluster */
} gen_cfg;

/* simple grid hash for the separation test */
typedef struct { int64_t cx, cy; int head; int used; } cell_t;
typedef struct { cell_t* cells; int ncell; double* re; double* im; int* next; int n; double g; } grid_t;

static uint64_t hkey(int64_t cx, int64_t cy) {
  uint64_t h = (uint64_t)cx * 0x9E3779B97F4A7C15ull ^ ((uint64_t)cy + 0x632BE59BD9B4E019ull) * 0xBF58476D1CE4E5B9ull;
  return h ^ (h >> 31);
}
static cell_t* grid_cell(grid_t* G, int64_t cx, int64_t cy, int create) {
  uint64_t h = hkey(cx, cy) % (uint64_t)G->ncell;
  for (;;) {
    cell_t* c = &G->cells[h];
    if (!c->used) {
      if (!create) return NULL;
      c->used = 1; c->cx = cx; c->cy = cy; c->head = -1;
      return c;
    }
    if (c->cx == cx && c->cy == cy) return c;
    h = (h + 1) % (uint64_t)G->ncell;
  }
}
static int grid_ok(grid_t* G, double re, double im) {
  int64_t cx = (int64_t)floor(re / G->g), cy = (int64_t)floor(im / G->g);
  for (int64_t dx = -1; dx <= 1; ++dx)
    for (int64_t dy = -1; dy <= 1; ++dy) {
      cell_t* c = grid_cell(G, cx + dx, cy + dy, 0);
      if (!c) continue;
      for (int q = c->head; q >= 0; q = G->next[q])
        if (hypot(G->re[q] - re, G->im[q] - im) < G->g) return 0;
    }
  return 1;
}
static void grid_add(grid_t* G, double re, double im) {
  int64_t cx = (int64_t)floor(re / G->g), cy = (int64_t)floor(im / G->g);
  cell_t* c = grid_cell(G, cx, cy, 1);
  G->re[G->n] = re; G->im[G->n] = im; G->next[G->n] = c->head; c->head = G->n; G->n++;
}

/* Diagonal-block values.  kinds[p] in {1,2}; vals[8p..8p+6] = (s | a,b,c), t | t1,t2 */
static void draw_block(const gen_cfg* g, uint64_t seed, int p, int kind, uint32_t attempt,
                       double* v) {
  double u[2], w[2], z[2];
  uni2(seed, TAG_DIAG, (uint64_t)p, attempt * 3 + 0, u);
  if (kind == 1) {
    v[0] = -1.0 + 2.0 * u[0];   /* s */
    v[1] = 0.5 + u[1];          /* t */
  } else {
    uni2(seed, TAG_DIAG, (uint64_t)p, attempt * 3 + 1, w);
    uni2(seed, TAG_DIAG, (uint64_t)p, attempt * 3 + 2, z);
    v[0] = -1.0 + 2.0 * u[0];   /* a */
    v[1] = 0.1 + 0.9 * u[1];    /* b */
    v[2] = 0.1 + 0.9 * w[0];    /* c */
    v[3] = 0.5 + w[1];          /* t1 */
    v[4] = 0.5 + z[0];          /* t2 */
  }
  (void)g;
}

/* planted eigenvalue(s) of a block (generator bookkeeping, closed form of the recipe) */
static void block_lambda(int kind, const double* v, double* re, double* im) {
  if (kind == 1) { *re = v[0] / v[1]; *im = 0.0; }
  else { *re = v[0] / v[3]; *im = sqrt(v[1] * v[2] / (v[3] * v[4])); }
}

/*
 * zzg_generate: fills S, T (column-major, m x m, leading dims lds, ldt) and, if not NULL,
 * lam_re[m], lam_im[m] with the planted eigenvalue of each row (+Im on the first row of a
 * pair, -Im on the second; inf for infinite eigenvalues).  Returns the number of reseeds /
 * redraws used (>= 0) or -1 on failure (separation not reachable, bad arguments, no memory).
 */
long zzg_generate(int m, int n2, double var_off, unsigned long long seed0, int gap_mode,
                  double gap, int n_zero, int n_inf, double stress_frac, int stress_tile,
                  double stress_scale, int cluster, double cluster_gap, double* S, long lds,
                  double* T, long ldt, double* lam_re, double* lam_im, int nthreads) {
  if (m < 0 || n2 < 0 || 2 * n2 > m || lds < (m > 1 ? m : 1) || ldt < (m > 1 ? m : 1)) return -1;
  gen_cfg g = {m, n2, var_off, seed0, gap_mode, gap, n_zero, n_inf, stress_frac, stress_tile,
               stress_scale, cluster, cluster_gap};
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  int nb = m - n2;
  int* kinds = (int*)malloc(sizeof(int) * (size_t)(nb > 0 ? nb : 1));
  int* start = (int*)malloc(sizeof(int) * (size_t)(nb > 0 ? nb : 1));
  double* vals = (double*)malloc(sizeof(double) * 8 * (size_t)(nb > 0 ? nb : 1));
  int* special = (int*)calloc((size_t)(nb > 0 ? nb : 1), sizeof(int)); /* 1 zero, 2 inf */
  double* clus = NULL;
  long redraws = 0;
  if (!kinds || !start || !vals || !special) { redraws = -1; goto out; }
  for (long attempt_pencil = 0;; ++attempt_pencil) {
    uint64_t seed = gap_mode == 1 ? seed0 * 1000ull + (uint64_t)attempt_pencil : seed0;
    /* block kinds in random order: Fisher-Yates over [2]*n2 + [1]*(nb-n2) */
    for (int p = 0; p < nb; ++p) kinds[p] = p < n2 ? 2 : 1;
    for (int p = nb - 1; p > 0; --p) {
      double u[2];
      uni2(seed, TAG_PERM, (uint64_t)p, 0, u);
      int q = (int)(u[0] * (double)(p + 1));
      if (q > p) q = p;
      int t = kinds[p]; kinds[p] = kinds[q]; kinds[q] = t;
    }
    for (int p = 0, r = 0; p < nb; ++p) { start[p] = r; r += kinds[p]; }
    /* special 1x1 blocks (zero / infinite eigenvalues): partial shuffle of the 1x1 list */
    memset(special, 0, sizeof(int) * (size_t)nb);
    {
      int n1 = nb - n2, k = 0;
      int* ones = (int*)malloc(sizeof(int) * (size_t)(n1 > 0 ? n1 : 1));
      for (int p = 0; p < nb; ++p) if (kinds[p] == 1) ones[k++] = p;
      int want = n_zero + n_inf;
      if (want > n1) want = n1;
      for (int i = 0; i < want; ++i) {
        double u[2];
        uni2(seed, TAG_SPECIAL, (uint64_t)i, 0, u);
        int q = i + (int)(u[0] * (double)(n1 - i));
        if (q >= n1) q = n1 - 1;
        int t = ones[i]; ones[i] = ones[q]; ones[q] = t;
        special[ones[i]] = i < n_zero ? 1 : 2;
      }
      /* clustered real spectrum (stress): real blocks in random order, clusters of size */
      if (cluster > 0) {
        int ncl = (n1 + cluster - 1) / cluster;
        clus = (double*)malloc(sizeof(double) * (size_t)(ncl > 0 ? ncl : 1));
        for (int c = 0; c < ncl; ++c) {
          double u[2];
          uni2(seed, TAG_CLUS, (uint64_t)c, 1, u);
          clus[c] = -1.5 + 3.0 * u[0];
        }
        for (int i = n1 - 1; i > 0; --i) {
          double u[2];
          uni2(seed, TAG_CLUS, (uint64_t)i, 0, u);
          int q = (int)(u[0] * (double)(i + 1));
          if (q > i) q = i;
          int t = ones[i]; ones[i] = ones[q]; ones[q] = t;
        }
        for (int i = 0; i < n1; ++i) {
          int p = ones[i];
          double u[2];
          draw_block(&g, seed, p, 1, 0, vals + 8 * (size_t)p);
          uni2(seed, TAG_CLUS, (uint64_t)p, 2, u);
          double t = 0.5 + u[0];
          double lam = clus[i / cluster] + (double)(i % cluster) * cluster_gap;
          vals[8 * (size_t)p] = lam * t;
          vals[8 * (size_t)p + 1] = t;
        }
      }
      free(ones);
    }
    /* draw the blocks; per-eigenvalue redraw (gap_mode 2) against all earlier eigenvalues */
    grid_t G = {0};
    if (gap_mode == 2) {
      G.ncell = 4 * m + 16;
      G.cells = (cell_t*)calloc((size_t)G.ncell, sizeof(cell_t));
      G.re = (double*)malloc(sizeof(double) * (size_t)(m + 1));
      G.im = (double*)malloc(sizeof(double) * (size_t)(m + 1));
      G.next = (int*)malloc(sizeof(int) * (size_t)(m + 1));
      G.g = gap;
    }
    int fail = 0;
    for (int p = 0; p < nb && !fail; ++p) {
      double* v = vals + 8 * (size_t)p;
      int fixed = (special[p] != 0) || (cluster > 0 && kinds[p] == 1);
      for (uint32_t att = 0;; ++att) {
        if (!fixed) draw_block(&g, seed, p, kinds[p], att, v);
        if (special[p] == 1) { draw_block(&g, seed, p, 1, att, v); v[0] = 0.0; }
        if (special[p] == 2) { draw_block(&g, seed, p, 1, att, v); v[1] = 0.0; }
        if (gap_mode != 2 || special[p] == 2) break;
        double re, im;
        block_lambda(kinds[p], v, &re, &im);
        int ok = grid_ok(&G, re, im) && (im == 0.0 || (2.0 * im >= gap && grid_ok(&G, re, -im)));
        if (ok || fixed) {
          grid_add(&G, re, im);
          if (im != 0.0) grid_add(&G, re, -im);
          break;
        }
        redraws++;
        if (att > 100000) { fail = 1; break; }
      }
    }
    free(G.cells); free(G.re); free(G.im); free(G.next);
    free(clus); clus = NULL;
    if (fail) { redraws = -1; goto out; }
    if (gap_mode == 1) {
      /* whole-pencil reseed until the min pairwise distance over all m eigenvalues >= gap */
      double* re = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
      double* im = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
      int k = 0;
      for (int p = 0; p < nb; ++p) {
        if (special[p] == 2) continue;
        double r0, i0;
        block_lambda(kinds[p], vals + 8 * (size_t)p, &r0, &i0);
        re[k] = r0; im[k++] = i0;
        if (kinds[p] == 2) { re[k] = r0; im[k++] = -i0; }
      }
      double mind = INFINITY;
      for (int i = 0; i < k; ++i)
        for (int j = i + 1; j < k; ++j) {
          double d = hypot(re[i] - re[j], im[i] - im[j]);
          if (d < mind) mind = d;
        }
      free(re); free(im);
      if (mind < gap) {
        redraws++;
        if (attempt_pencil > 10000) { redraws = -1; goto out; }
        continue;
      }
    }
    /* fill S and T */
    int* rowblk = (int*)malloc(sizeof(int) * (size_t)(m > 0 ? m : 1));
    for (int p = 0; p < nb; ++p)
      for (int q = 0; q < kinds[p]; ++q) rowblk[start[p] + q] = p;
    /* stress tiles on a fixed generator grid (strictly-upper tiles I < J) */
    unsigned char* big = NULL;
    int ntile = 0;
    if (stress_frac > 0 && stress_tile > 0) {
      ntile = (m + stress_tile - 1) / stress_tile;
      long nup = (long)ntile * (ntile - 1) / 2;
      long want = (long)llround(stress_frac * (double)nup);
      big = (unsigned char*)calloc((size_t)ntile * (size_t)(ntile > 0 ? ntile : 1), 1);
      long* ids = (long*)malloc(sizeof(long) * (size_t)(nup > 0 ? nup : 1));
      for (long i = 0; i < nup; ++i) ids[i] = i;
      for (long i = 0; i < want; ++i) {
        double u[2];
        uni2(seed, TAG_TILES, (uint64_t)i, 0, u);
        long q = i + (long)(u[0] * (double)(nup - i));
        if (q >= nup) q = nup - 1;
        long t = ids[i]; ids[i] = ids[q]; ids[q] = t;
        /* decode linear strictly-upper tile index -> (I, J), column-major over J */
        long id = ids[i], J = 1;
        while (id >= J) { id -= J; J++; }
        big[(size_t)J * ntile + (size_t)id] = 1;
      }
      free(ids);
    }
    double sd = sqrt(var_off);
#pragma omp parallel for schedule(dynamic, 16)
    for (int j = 0; j < m; ++j) {
      double* sc = S + (size_t)j * (size_t)lds;
      double* tc = T + (size_t)j * (size_t)ldt;
      int pj = rowblk[j];
      for (int i = 0; i < m; ++i) {
        double sv = 0.0, tv = 0.0;
        if (i < j) {
          int pi = rowblk[i];
          if (pi != pj) {
            uint64_t idx = (uint64_t)i + (uint64_t)j * (uint64_t)m;
            sv = sd * normal(seed, TAG_OFFS, idx);
            tv = sd * normal(seed, TAG_OFFT, idx);
            if (big && big[(size_t)(j / stress_tile) * ntile + (size_t)(i / stress_tile)]) {
              sv *= stress_scale;
              tv *= stress_scale;
            }
          }
        }
        sc[i] = sv;
        tc[i] = tv;
      }
    }
    free(big);
    for (int p = 0; p < nb; ++p) {
      int j = start[p];
      const double* v = vals + 8 * (size_t)p;
      double re, im;
      if (kinds[p] == 1) {
        S[(size_t)j * lds + j] = v[0];
        T[(size_t)j * ldt + j] = v[1];
        block_lambda(1, v, &re, &im);
        if (v[1] == 0.0) re = INFINITY;
        if (lam_re) { lam_re[j] = re; lam_im[j] = 0.0; }
      } else {
        double a = v[0], b = v[1], c = v[2], t1 = v[3], t2 = v[4];
        S[(size_t)j * lds + j] = a;
        S[(size_t)j * lds + j + 1] = -c;
        S[(size_t)(j + 1) * lds + j] = b;
        S[(size_t)(j + 1) * lds + j + 1] = a * t2 / t1;
        T[(size_t)j * ldt + j] = t1;
        T[(size_t)(j + 1) * ldt + j] = 0.0;
        T[(size_t)(j + 1) * ldt + j + 1] = t2;
        block_lambda(2, v, &re, &im);
        if (lam_re) { lam_re[j] = re; lam_im[j] = im; lam_re[j + 1] = re; lam_im[j + 1] = -im; }
      }
    }
    free(rowblk);
    break;
  }
out:
  free(kinds); free(start); free(vals); free(special); free(clus);
  return redraws;
}
