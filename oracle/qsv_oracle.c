/*
 * CPU oracle, plain-C restatement of the reference kernels for large n.
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/ and by bench.py's cpu-baseline
 * leg through ctypes, never by the product package.  It exists because the
 * numpy restatement (oracle/qsim_oracle.py) needs ~63-80 B/amp and several
 * seconds per gate at 28 qubits, which is too slow
 * for parity at the benchmark sizes.
 *
 * Algorithm (cited into /root/reference/pkg/src/qsimcore):
 *   - cosets: B0 = counter with zero bits inserted at the fixed positions
 *     (kernels.py:28-39), B1 = 2^m offsets with counter bit j -> targets[j]
 *     (kernels.py:42-52), control-value shift (kernels.py:55-56, 73-76);
 *   - dense: per coset gather 2^m amps, out[z] = sum_w K[z][w] in[w],
 *     scatter (kernels.py:79-138);
 *   - diagonal: amp *= d[sub(idx)] (kernels.py:155-173);
 *   - Pauli / rotation: (P psi)_x = i^ny (-1)^popc(src & zy) psi_src with
 *     src = x ^ xmask, rot = cos(a/2) psi + i sin(a/2) P psi
 *     (kernels.py:188-235);
 *   - expectation: sum_t c_t <psi|P_t|psi> (observable.py:99-104).
 * Complex products are written out as real arithmetic in numpy's order and
 * the file is compiled with -ffp-contract=off, so the 1-qubit and rotation
 * paths reproduce the numpy oracle bit for bit.
 *
 * Build: see oracle/Makefile (gcc -O2 -fopenmp -ffp-contract=off).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef struct { double re, im; } cplx;

static inline cplx cmul(cplx a, cplx b) {
  cplx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}
static inline cplx cadd(cplx a, cplx b) {
  cplx r = {a.re + b.re, a.im + b.im};
  return r;
}

/* insert a zero bit at every position of the ascending list `pos` */
static inline uint64_t widen(uint64_t k, const int* pos, int np) {
  for (int i = 0; i < np; ++i) {
    uint64_t low = k & ((1ULL << pos[i]) - 1ULL);
    k = ((k ^ low) << 1) | low;
  }
  return k;
}

static void sort_ints(int* v, int n) {
  for (int i = 1; i < n; ++i) {
    int x = v[i], j = i - 1;
    while (j >= 0 && v[j] > x) { v[j + 1] = v[j]; --j; }
    v[j + 1] = x;
  }
}

/* dense 2^m x 2^m (row-major, interleaved complex) on targets with controls */
int oracle_apply_dense(double* amps_, int n, const int* targets, int m,
                       const double* mat_, const int* cq, const int* cv, int nc) {
  cplx* a = (cplx*)amps_;
  const cplx* K = (const cplx*)mat_;
  int fixed[64];
  int nf = 0;
  uint64_t shift = 0;
  for (int i = 0; i < m; ++i) fixed[nf++] = targets[i];
  for (int i = 0; i < nc; ++i) { fixed[nf++] = cq[i]; if (cv[i]) shift |= 1ULL << cq[i]; }
  sort_ints(fixed, nf);
  const uint64_t dim = 1ULL << m;
  uint64_t* offs = (uint64_t*)malloc(sizeof(uint64_t) * dim);
  for (uint64_t z = 0; z < dim; ++z) {
    uint64_t o = 0;
    for (int j = 0; j < m; ++j) if ((z >> j) & 1ULL) o |= 1ULL << targets[j];
    offs[z] = o;
  }
  const int64_t ncos = (int64_t)(1ULL << (n - nf));
#pragma omp parallel
  {
    cplx* in = (cplx*)malloc(sizeof(cplx) * dim);
#pragma omp for schedule(static)
    for (int64_t k = 0; k < ncos; ++k) {
      uint64_t base = widen((uint64_t)k, fixed, nf) + shift;
      for (uint64_t w = 0; w < dim; ++w) in[w] = a[base + offs[w]];
      for (uint64_t z = 0; z < dim; ++z) {
        cplx acc = cmul(K[z * dim], in[0]);
        for (uint64_t w = 1; w < dim; ++w) acc = cadd(acc, cmul(K[z * dim + w], in[w]));
        a[base + offs[z]] = acc;
      }
    }
    free(in);
  }
  free(offs);
  return 0;
}

int oracle_apply_diag(double* amps_, int n, const int* targets, int m,
                      const double* diag_, const int* cq, const int* cv, int nc) {
  cplx* a = (cplx*)amps_;
  const cplx* d = (const cplx*)diag_;
  int fixed[64];
  uint64_t shift = 0;
  for (int i = 0; i < nc; ++i) { fixed[i] = cq[i]; if (cv[i]) shift |= 1ULL << cq[i]; }
  sort_ints(fixed, nc);
  const int64_t cnt = (int64_t)(1ULL << (n - nc));
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < cnt; ++k) {
    uint64_t x = widen((uint64_t)k, fixed, nc) + shift;
    uint64_t sub = 0;
    for (int j = 0; j < m; ++j) sub |= ((x >> targets[j]) & 1ULL) << j;
    a[x] = cmul(a[x], d[sub]);
  }
  return 0;
}

static void masks(const int* targets, const int* ids, int m,
                  uint64_t* xm, uint64_t* zm, int* ny) {
  *xm = 0; *zm = 0; *ny = 0;
  for (int i = 0; i < m; ++i) {
    if (ids[i] == 1 || ids[i] == 2) *xm |= 1ULL << targets[i];
    if (ids[i] == 2 || ids[i] == 3) *zm |= 1ULL << targets[i];
    if (ids[i] == 2) ++*ny;
  }
}

static const cplx IPOW[4] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};

/* (P psi)_x for one x */
static inline cplx pauli_elem(const cplx* a, uint64_t x, uint64_t xm, uint64_t zm, int ny) {
  uint64_t src = x ^ xm;
  cplx v = a[src];
  if (__builtin_popcountll(src & zm) & 1) { v.re = -v.re; v.im = -v.im; }
  if (ny % 4) v = cmul(v, IPOW[ny % 4]);
  return v;
}

/* exp(i angle P / 2), uncontrolled (controlled rotations go through dense) */
int oracle_apply_pauli_rot(double* amps_, int n, const int* targets, const int* ids,
                           int m, double angle) {
  cplx* a = (cplx*)amps_;
  uint64_t xm, zm;
  int ny;
  masks(targets, ids, m, &xm, &zm, &ny);
  const double c = cos(angle / 2), s = sin(angle / 2);
  const int64_t dim = (int64_t)(1ULL << n);
  if (!xm) {
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < dim; ++x) {
      cplx p = pauli_elem(a, (uint64_t)x, 0, zm, ny);
      cplx v = a[x];
      a[x].re = v.re * c + (-s * p.im);
      a[x].im = v.im * c + (s * p.re);
    }
    return 0;
  }
  int pivot = 63 - __builtin_clzll(xm);
  const int64_t half = dim >> 1;
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < half; ++k) {
    uint64_t i = widen((uint64_t)k, &pivot, 1);
    uint64_t j = i ^ xm;
    cplx pi = pauli_elem(a, i, xm, zm, ny);
    cplx pj = pauli_elem(a, j, xm, zm, ny);
    cplx vi = a[i], vj = a[j];
    a[i].re = vi.re * c + (-s * pi.im);
    a[i].im = vi.im * c + (s * pi.re);
    a[j].re = vj.re * c + (-s * pj.im);
    a[j].im = vj.im * c + (s * pj.re);
  }
  return 0;
}

int oracle_apply_pauli(double* amps_, int n, const int* targets, const int* ids, int m) {
  cplx* a = (cplx*)amps_;
  uint64_t xm, zm;
  int ny;
  masks(targets, ids, m, &xm, &zm, &ny);
  const int64_t dim = (int64_t)(1ULL << n);
  if (!xm) {
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < dim; ++x) a[x] = pauli_elem(a, (uint64_t)x, 0, zm, ny);
    return 0;
  }
  int pivot = 63 - __builtin_clzll(xm);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < (dim >> 1); ++k) {
    uint64_t i = widen((uint64_t)k, &pivot, 1);
    uint64_t j = i ^ xm;
    cplx pi = pauli_elem(a, i, xm, zm, ny);
    cplx pj = pauli_elem(a, j, xm, zm, ny);
    a[i] = pi;
    a[j] = pj;
  }
  return 0;
}

/* <bra| P |ket> for one Pauli product, summed in double */
int oracle_pauli_term(const double* bra_, const double* ket_, int n, const int* targets,
                      const int* ids, int m, double out[2]) {
  const cplx* b = (const cplx*)bra_;
  const cplx* k = (const cplx*)ket_;
  uint64_t xm, zm;
  int ny;
  masks(targets, ids, m, &xm, &zm, &ny);
  const int64_t dim = (int64_t)(1ULL << n);
  double re = 0, im = 0;
#pragma omp parallel for reduction(+ : re, im) schedule(static)
  for (int64_t x = 0; x < dim; ++x) {
    cplx p = pauli_elem(k, (uint64_t)x, xm, zm, ny);
    re += b[x].re * p.re + b[x].im * p.im;
    im += b[x].re * p.im - b[x].im * p.re;
  }
  out[0] = re;
  out[1] = im;
  return 0;
}

int oracle_norm2(const double* amps_, int n, double* out) {
  const cplx* a = (const cplx*)amps_;
  const int64_t dim = (int64_t)(1ULL << n);
  double s = 0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (int64_t x = 0; x < dim; ++x) s += a[x].re * a[x].re + a[x].im * a[x].im;
  *out = s;
  return 0;
}
