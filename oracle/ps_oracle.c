/*
 * ps_oracle.c — CPU restatement of the reference's stencil arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker the GPU path is compared against
 * (tests/, __graft_entry__.smoke(), bench.py's cpu_baseline / --impl reference legs).
 * The product (paper_1904_04048_b200, libps.so) never links, loads or calls it.
 *
 * It restates, on the reference's own dense (rows x cols) arrays, the operation
 * sequence of poisson_stencils/simulator.py (pkg/src/poisson_stencils/):
 *   _apply_evaluated            simulator.py:147-163   (Dirichlet slices :151-155,
 *                                                       periodic np.roll :156-162)
 *   _alias_edges                simulator.py:135-138
 *   first_step                  simulator.py:166-180
 *   _two_step_evaluated         simulator.py:183-191   (re-pinned ring :185-190)
 * Per point: acc = +0.0; for each tap in table order acc = fl(acc + fl(c * u[nb]));
 * no FMA (built with -ffp-contract=off).  float32 fields follow numpy's promotion:
 * fl32(fl32(c) * u) added into a float64 accumulator, stored to float32, float32
 * subtract / add (simulator.py:150-154, 179, 184).  The "native" f32 contract is the
 * GPU's own (PS_ARITH_NATIVE, not a reference path): taps folded in with fmaf() in
 * table order, float32 accumulator.
 *
 * Generalisation beyond the reference: the Dirichlet ring width is
 * a parameter (reference: 1, simulator.py:98-102); at ring = 1 the arithmetic is the
 * reference's exactly.  Pinned by tests/golden (generated from the live reference).
 *
 * Rows are independent, so the loops are OpenMP-parallel over rows; results do not
 * depend on the thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <math.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { ORA_F64 = 0, ORA_F32 = 1 };
enum { ORA_DIRICHLET = 0, ORA_PERIODIC = 1 };
enum { ORA_REF = 0, ORA_NATIVE = 1 };

typedef struct {
  int n;
  const int* q1;
  const int* q2;
  const double* c;
} tab_t;

static int64_t wrap(int64_t x, int64_t n) {
  x %= n;
  return x < 0 ? x + n : x;
}

/* acc over row i for columns [j0, j1) into accd (f64 contract) — per point, taps in
 * table order.  get(i, j) addressing is resolved by the caller through (base, pitch,
 * periodic core sizes). */
static void row_acc_f64(const tab_t* t, const double* u, int64_t cols, int per, int64_t n1,
                        int64_t n2, int64_t i, int64_t j0, int64_t j1, double* acc) {
  for (int64_t j = j0; j < j1; ++j) acc[j - j0] = 0.0;
  for (int s = 0; s < t->n; ++s) {
    const double c = t->c[s];
    if (per) {
      const double* row = u + wrap(i + t->q1[s], n1) * cols;
      for (int64_t j = j0; j < j1; ++j) acc[j - j0] = acc[j - j0] + c * row[wrap(j + t->q2[s], n2)];
    } else {
      const double* row = u + (i + t->q1[s]) * cols + t->q2[s];
      for (int64_t j = j0; j < j1; ++j) acc[j - j0] = acc[j - j0] + c * row[j];
    }
  }
}

static void row_acc_f32ref(const tab_t* t, const float* u, int64_t cols, int per, int64_t n1,
                           int64_t n2, int64_t i, int64_t j0, int64_t j1, double* acc) {
  for (int64_t j = j0; j < j1; ++j) acc[j - j0] = 0.0;
  for (int s = 0; s < t->n; ++s) {
    const float c = (float)t->c[s];
    if (per) {
      const float* row = u + wrap(i + t->q1[s], n1) * cols;
      for (int64_t j = j0; j < j1; ++j) {
        const float p = c * row[wrap(j + t->q2[s], n2)];
        acc[j - j0] = acc[j - j0] + (double)p;
      }
    } else {
      const float* row = u + (i + t->q1[s]) * cols + t->q2[s];
      for (int64_t j = j0; j < j1; ++j) {
        const float p = c * row[j];
        acc[j - j0] = acc[j - j0] + (double)p;
      }
    }
  }
}

/* GPU "native" f32 contract (not a reference path): acc = fmaf(c, u, acc) per tap in
 * table order from +0.0 — one correctly rounded fused multiply-add per tap. */
static void row_acc_f32nat(const tab_t* t, const float* u, int64_t cols, int per, int64_t n1,
                           int64_t n2, int64_t i, int64_t j0, int64_t j1, float* acc) {
  for (int64_t j = j0; j < j1; ++j) acc[j - j0] = 0.0f;
  for (int s = 0; s < t->n; ++s) {
    const float c = (float)t->c[s];
    if (per) {
      const float* row = u + wrap(i + t->q1[s], n1) * cols;
      for (int64_t j = j0; j < j1; ++j)
        acc[j - j0] = fmaf(c, row[wrap(j + t->q2[s], n2)], acc[j - j0]);
    } else {
      const float* row = u + (i + t->q1[s]) * cols + t->q2[s];
      for (int64_t j = j0; j < j1; ++j) acc[j - j0] = fmaf(c, row[j], acc[j - j0]);
    }
  }
}

/* Row range helpers.  Dirichlet: rows/cols include the ring; interior rows/cols are
 * [ring, rows-ring).  Periodic: rows = n1+1, cols = n2+1 (alias row/col included). */

static int check(int bc, int ring, int64_t rows, int64_t cols, const tab_t* t) {
  if (rows < 1 || cols < 1) return 2;
  if (t->n < 1) return 3;
  int r = 0;
  for (int s = 0; s < t->n; ++s) {
    int a = abs(t->q1[s]), b = abs(t->q2[s]);
    if (a > r) r = a;
    if (b > r) r = b;
  }
  if (bc == ORA_DIRICHLET) {
    if (ring < r) return 4;
    if (2 * (int64_t)ring > rows || 2 * (int64_t)ring > cols) return 2;
  } else {
    if (rows < 2 || cols < 2) return 2;
  }
  return 0;
}

/* two_step over rows [row_lo, row_hi) of the output (row_hi <= 0 means all rows). */
int ora_two_step(int dtype, int arith, int bc, int ring, int64_t rows, int64_t cols, int ntaps,
                 const int* q1, const int* q2, const double* c, const void* uk,
                 const void* ukm1, void* out, int64_t row_lo, int64_t row_hi, int nthreads) {
  tab_t t = {ntaps, q1, q2, c};
  int st = check(bc, ring, rows, cols, &t);
  if (st) return st;
  if (dtype != ORA_F64 && dtype != ORA_F32) return 1;
  if (row_hi <= 0 || row_hi > rows) row_hi = rows;
  if (row_lo < 0) row_lo = 0;
  const int per = bc == ORA_PERIODIC;
  const int64_t n1 = per ? rows - 1 : rows, n2 = per ? cols - 1 : cols;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
  {
    double* accd = (double*)malloc(sizeof(double) * (size_t)(cols + 1));
    float* accf = (float*)malloc(sizeof(float) * (size_t)(cols + 1));
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
    for (int64_t i = row_lo; i < row_hi; ++i) {
      if (!per) {
        const int ring_row = i < ring || i >= rows - ring;
        if (dtype == ORA_F64) {
          double* o = (double*)out + i * cols;
          const double* km = (const double*)ukm1 + i * cols;
          if (ring_row) {
            for (int64_t j = 0; j < cols; ++j) o[j] = 0.0;
            continue;
          }
          row_acc_f64(&t, (const double*)uk, cols, 0, n1, n2, i, ring, cols - ring, accd);
          for (int64_t j = 0; j < ring; ++j) o[j] = 0.0, o[cols - 1 - j] = 0.0;
          for (int64_t j = ring; j < cols - ring; ++j) o[j] = accd[j - ring] - km[j];
        } else {
          float* o = (float*)out + i * cols;
          const float* km = (const float*)ukm1 + i * cols;
          if (ring_row) {
            for (int64_t j = 0; j < cols; ++j) o[j] = 0.0f;
            continue;
          }
          for (int64_t j = 0; j < ring; ++j) o[j] = 0.0f, o[cols - 1 - j] = 0.0f;
          if (arith == ORA_NATIVE) {
            row_acc_f32nat(&t, (const float*)uk, cols, 0, n1, n2, i, ring, cols - ring, accf);
            for (int64_t j = ring; j < cols - ring; ++j) o[j] = accf[j - ring] - km[j];
          } else {
            row_acc_f32ref(&t, (const float*)uk, cols, 0, n1, n2, i, ring, cols - ring, accd);
            for (int64_t j = ring; j < cols - ring; ++j) o[j] = (float)accd[j - ring] - km[j];
          }
        }
      } else {
        /* core row ic = i mod n1 supplies the acc; the alias row n1 reuses row 0's acc,
         * the alias column reuses column 0's acc (simulator.py:135-138, 184). */
        const int64_t ic = i == n1 ? 0 : i;
        if (dtype == ORA_F64) {
          double* o = (double*)out + i * cols;
          const double* km = (const double*)ukm1 + i * cols;
          row_acc_f64(&t, (const double*)uk, cols, 1, n1, n2, ic, 0, n2, accd);
          for (int64_t j = 0; j < n2; ++j) o[j] = accd[j] - km[j];
          o[n2] = accd[0] - km[n2];
        } else {
          float* o = (float*)out + i * cols;
          const float* km = (const float*)ukm1 + i * cols;
          if (arith == ORA_NATIVE) {
            row_acc_f32nat(&t, (const float*)uk, cols, 1, n1, n2, ic, 0, n2, accf);
            for (int64_t j = 0; j < n2; ++j) o[j] = accf[j] - km[j];
            o[n2] = accf[0] - km[n2];
          } else {
            row_acc_f32ref(&t, (const float*)uk, cols, 1, n1, n2, ic, 0, n2, accd);
            for (int64_t j = 0; j < n2; ++j) o[j] = (float)accd[j] - km[j];
            o[n2] = (float)accd[0] - km[n2];
          }
        }
      }
    }
    free(accd);
    free(accf);
  }
  return 0;
}

int ora_first_step(int dtype, int arith, int bc, int ring, int64_t rows, int64_t cols,
                   int ntu, const int* q1u, const int* q2u, const double* cu, int ntv,
                   const int* q1v, const int* q2v, const double* cv, double tau,
                   const void* u0, const void* v0, void* out, int nthreads) {
  tab_t tu = {ntu, q1u, q2u, cu}, tv = {ntv, q1v, q2v, cv};
  int st = check(bc, ring, rows, cols, &tu);
  if (st) return st;
  if ((st = check(bc, ring, rows, cols, &tv))) return st;
  if (dtype != ORA_F64 && dtype != ORA_F32) return 1;
  const int per = bc == ORA_PERIODIC;
  const int64_t n1 = per ? rows - 1 : rows, n2 = per ? cols - 1 : cols;
  const int64_t jlo = per ? 0 : ring, jhi = per ? n2 : cols - ring;
  const float tauf = (float)tau;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
  {
    double* au = (double*)malloc(sizeof(double) * (size_t)(cols + 1));
    double* av = (double*)malloc(sizeof(double) * (size_t)(cols + 1));
    float* fu = (float*)malloc(sizeof(float) * (size_t)(cols + 1));
    float* fv = (float*)malloc(sizeof(float) * (size_t)(cols + 1));
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
    for (int64_t i = 0; i < rows; ++i) {
      const int ring_row = !per && (i < ring || i >= rows - ring);
      const int64_t ic = (per && i == n1) ? 0 : i;
      if (dtype == ORA_F64) {
        double* o = (double*)out + i * cols;
        for (int64_t j = 0; j < cols; ++j) o[j] = 0.0;
        if (ring_row) continue;
        row_acc_f64(&tu, (const double*)u0, cols, per, n1, n2, ic, jlo, jhi, au);
        row_acc_f64(&tv, (const double*)v0, cols, per, n1, n2, ic, jlo, jhi, av);
        for (int64_t j = jlo; j < jhi; ++j) o[j] = au[j - jlo] + tau * av[j - jlo];
        if (per) o[n2] = o[0];
      } else {
        float* o = (float*)out + i * cols;
        for (int64_t j = 0; j < cols; ++j) o[j] = 0.0f;
        if (ring_row) continue;
        if (arith == ORA_NATIVE) {
          row_acc_f32nat(&tu, (const float*)u0, cols, per, n1, n2, ic, jlo, jhi, fu);
          row_acc_f32nat(&tv, (const float*)v0, cols, per, n1, n2, ic, jlo, jhi, fv);
          for (int64_t j = jlo; j < jhi; ++j) o[j] = fu[j - jlo] + tauf * fv[j - jlo];
        } else {
          row_acc_f32ref(&tu, (const float*)u0, cols, per, n1, n2, ic, jlo, jhi, au);
          row_acc_f32ref(&tv, (const float*)v0, cols, per, n1, n2, ic, jlo, jhi, av);
          for (int64_t j = jlo; j < jhi; ++j) {
            const float a = (float)au[j - jlo];
            const float b = tauf * (float)av[j - jlo];
            o[j] = a + b;
          }
        }
        if (per) o[n2] = o[0];
      }
    }
    free(au);
    free(av);
    free(fu);
    free(fv);
  }
  return 0;
}

/* nsteps two-step updates rotating three caller buffers (lvl[newest] = u^k,
 * lvl[(newest+2)%3] = u^{k-1}); returns the index of the newest level via *newest. */
int ora_march(int dtype, int arith, int bc, int ring, int64_t rows, int64_t cols, int ntaps,
              const int* q1, const int* q2, const double* c, void* l0, void* l1, void* l2,
              int64_t nsteps, int* newest, int nthreads) {
  void* lvl[3] = {l0, l1, l2};
  int cur = *newest;
  for (int64_t k = 0; k < nsteps; ++k) {
    const int prev = (cur + 2) % 3, next = (cur + 1) % 3;
    int st = ora_two_step(dtype, arith, bc, ring, rows, cols, ntaps, q1, q2, c, lvl[cur],
                          lvl[prev], lvl[next], 0, 0, nthreads);
    if (st) return st;
    cur = next;
  }
  *newest = cur;
  return 0;
}

int ora_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
