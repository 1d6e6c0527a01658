/*
 * mpmm_oracle.c -- CPU restatement of the reference DD/QD kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may use it, and only as the checker.
 *
 * It restates the operation sequences of the reference's compiled kernel
 * module /root/reference/pkg/src/mpmm/_kernels.pyx (and its Python mirror
 * _kernels_py.py / ddqd.py / eft.py) in plain C.  The reference is compiled
 * with -O3 -ffp-contract=off -fno-fast-math (pkg/setup.py:9-11); this file
 * must be compiled with the same flags (see oracle/Makefile) so every
 * multiply and add rounds exactly as the reference's do.  TwoProd uses the
 * Veltkamp/Dekker split exactly like the reference (no FMA), so this oracle
 * is an independent check of the GPU's FMA-based TwoProd.
 *
 * Layout contract (reference matrix.py:20,43-48): a DD matrix is a
 * C-contiguous float64 array (rows, cols, 2), a QD matrix (rows, cols, 4).
 * Leading dimensions here are in ELEMENTS (one element = 2 or 4 doubles) so
 * the Strassen restatement can address quadrants without copies.
 *
 * Parity pinning: tests/test_oracle_golden.py checks these functions against
 * golden vectors produced by the reference itself (tests/golden/make_golden.py)
 * and, when present, against the reference kernels compiled into oracle/_ref.
 */
#include <stdint.h>
#include <string.h>

typedef int64_t i64;

/* eft.py:19 / _kernels.pyx:15 -- Veltkamp splitter 2^27 + 1 */
static const double SPLITTER = 134217729.0;
/* ddqd.py:28 / _kernels.pyx:16 -- compression passes for QD term sums */
#define QD_PASSES 4

/* eft.py:39-42 _split */
static inline void vsplit(double a, double *hi, double *lo) {
    double t = SPLITTER * a;
    double h = t - (t - a);
    *hi = h;
    *lo = a - h;
}

/* eft.py:45-49 _two_prod_raw == _kernels.pyx:19-29 _two_prod */
static inline double two_prod(double a, double b, double *err) {
    double p = a * b;
    double ah, al, bh, bl;
    vsplit(a, &ah, &al);
    vsplit(b, &bh, &bl);
    *err = ((ah * bh - p) + ah * bl + al * bh) + al * bl;
    return p;
}

/* eft.py:27-30 _two_sum_raw */
static inline double two_sum(double a, double b, double *err) {
    double s = a + b;
    double bb = s - a;
    *err = (a - (s - bb)) + (b - bb);
    return s;
}

/* eft.py:33-36 _quick_two_sum_raw */
static inline double quick_two_sum(double a, double b, double *err) {
    double s = a + b;
    *err = b - (s - a);
    return s;
}

/* ------------------------------------------------------------------------ */
/* double-double                                                            */
/* ------------------------------------------------------------------------ */

/* ddqd.py:63-70 dd_add == _kernels.pyx:189-204 _dd_add */
static inline void dd_add(double xh, double xl, double yh, double yl,
                          double *hi, double *lo) {
    double s2, t2, e;
    double s1 = two_sum(xh, yh, &s2);
    double t1 = two_sum(xl, yl, &t2);
    s2 = s2 + t1;
    s1 = quick_two_sum(s1, s2, &e);
    s2 = e + t2;
    *hi = quick_two_sum(s1, s2, lo);
}

/* ddqd.py:77-91 dd_mul with the shared splits of _kernels.pyx:140-171 */
static inline void dd_mul(double ah, double al, double bh, double bl,
                          double *ph, double *pl) {
    double e, e1, e2, r1, r2, w;
    double p = two_prod(ah, bh, &e);
    double p1 = two_prod(ah, bl, &e1);
    double p2 = two_prod(al, bh, &e2);
    double tail = (e1 + e2) + al * bl;
    double s = two_sum(p1, p2, &r1);
    s = two_sum(e, s, &r2);
    double losum = (r1 + r2) + tail;
    double hi = quick_two_sum(p, s, &w);
    w = w + losum;
    *ph = quick_two_sum(hi, w, pl);
}

/* One multiply-add c <- dd_add(c, dd_mul(a, b)): the k-loop body of
 * _kernels.pyx:135-184 (dd_block_cells) and :49-98 (dd_simple_rows). */
static inline void dd_madd(double *ch, double *cl, const double *a, const double *b) {
    double ph, pl;
    dd_mul(a[0], a[1], b[0], b[1], &ph, &pl);
    dd_add(*ch, *cl, ph, pl, ch, cl);
}

/* _kernels.pyx:36-100 dd_simple_rows: rows [i0, i1) of C, acc from (0, 0),
 * k ascending, C overwritten. */
void oracle_dd_simple_rows(const double *A, i64 lda, const double *B, i64 ldb,
                           double *C, i64 ldc, i64 l, i64 n, i64 i0, i64 i1) {
    for (i64 i = i0; i < i1; ++i)
        for (i64 j = 0; j < n; ++j) {
            double ch = 0.0, cl = 0.0;
            for (i64 k = 0; k < l; ++k)
                dd_madd(&ch, &cl, A + 2 * (i * lda + k), B + 2 * (k * ldb + j));
            C[2 * (i * ldc + j)] = ch;
            C[2 * (i * ldc + j) + 1] = cl;
        }
}

/* _kernels.pyx:103-186 dd_block_cells: cells [cell0, cell1) of the
 * ceil(m/n_min) x ceil(n/n_min) grid, accumulating INTO C (:133-134). */
void oracle_dd_block_cells(const double *A, i64 lda, const double *B, i64 ldb,
                           double *C, i64 ldc, i64 m, i64 l, i64 n, i64 n_min,
                           i64 cell0, i64 cell1) {
    i64 nb_cols = (n + n_min - 1) / n_min;
    i64 lb = (l + n_min - 1) / n_min;
    for (i64 cell = cell0; cell < cell1; ++cell) {
        i64 ib = cell / nb_cols, jb = cell - (cell / nb_cols) * nb_cols;
        i64 ilo = ib * n_min, ihi = ilo + n_min < m ? ilo + n_min : m;
        i64 jlo = jb * n_min, jhi = jlo + n_min < n ? jlo + n_min : n;
        for (i64 kb = 0; kb < lb; ++kb) {
            i64 klo = kb * n_min, khi = klo + n_min < l ? klo + n_min : l;
            for (i64 i = ilo; i < ihi; ++i)
                for (i64 j = jlo; j < jhi; ++j) {
                    double *c = C + 2 * (i * ldc + j);
                    double ch = c[0], cl = c[1];
                    for (i64 k = klo; k < khi; ++k)
                        dd_madd(&ch, &cl, A + 2 * (i * lda + k), B + 2 * (k * ldb + j));
                    c[0] = ch;
                    c[1] = cl;
                }
        }
    }
}

/* _kernels.pyx:207-230 dd_ewise_add / dd_ewise_sub over rows [i0, i1). */
void oracle_dd_ewise(const double *X, i64 ldx, const double *Y, i64 ldy,
                     double *O, i64 ldo, i64 cols, i64 i0, i64 i1, int subtract) {
    for (i64 i = i0; i < i1; ++i)
        for (i64 j = 0; j < cols; ++j) {
            const double *x = X + 2 * (i * ldx + j);
            const double *y = Y + 2 * (i * ldy + j);
            double yh = subtract ? -y[0] : y[0];
            double yl = subtract ? -y[1] : y[1];
            double hi, lo;
            dd_add(x[0], x[1], yh, yl, &hi, &lo);
            O[2 * (i * ldo + j)] = hi;
            O[2 * (i * ldo + j) + 1] = lo;
        }
}

/* ------------------------------------------------------------------------ */
/* quad-double                                                              */
/* ------------------------------------------------------------------------ */

/* ddqd.py:140-172 _renorm5 == _kernels.pyx:237-271 */
static void renorm5(double x0, double x1, double x2, double x3, double x4,
                    double out[4]) {
    double s, t;
    s = quick_two_sum(x3, x4, &x4);
    t = quick_two_sum(x2, s, &x3);
    s = quick_two_sum(x1, t, &x2);
    t = quick_two_sum(x0, s, &x1);
    double rest[4] = {x1, x2, x3, x4};
    out[0] = out[1] = out[2] = out[3] = 0.0;
    double acc = t;
    int k = 0;
    for (int idx = 0; idx < 4; ++idx) {
        double v = rest[idx];
        if (k == 3) {
            acc += v;
            continue;
        }
        double e;
        acc = quick_two_sum(acc, v, &e);
        if (e != 0.0) {
            out[k++] = acc;
            acc = e;
        }
    }
    out[k] = acc;
}

/* ddqd.py:175-193 _compress4 == _kernels.pyx:274-308: drop zero terms
 * (including -0.0), QD_PASSES error-free vector passes, tail sum, renorm5. */
static void compress4(const double *terms, int nterms, double out[4]) {
    double buf[24];
    int n = 0;
    for (int i = 0; i < nterms; ++i)
        if (terms[i] != 0.0) buf[n++] = terms[i];
    if (n == 0) {
        out[0] = out[1] = out[2] = out[3] = 0.0;
        return;
    }
    for (int p = 0; p < QD_PASSES; ++p) {
        double s = buf[0];
        for (int i = 1; i < n; ++i) s = two_sum(s, buf[i], &buf[i - 1]);
        buf[n - 1] = s;
    }
    if (n <= 4) {
        double w[4] = {0.0, 0.0, 0.0, 0.0};
        for (int i = 0; i < n; ++i) w[4 - n + i] = buf[i];
        renorm5(w[3], w[2], w[1], w[0], 0.0, out);
        return;
    }
    double tail = 0.0;
    for (int i = 0; i < n - 4; ++i) tail += buf[i];
    renorm5(buf[n - 1], buf[n - 2], buf[n - 3], buf[n - 4], tail, out);
}

/* _kernels.pyx:311-341 _qd_mul_add == ddqd.qd_add(cc, ddqd.qd_mul(x, y))
 * (ddqd.py:208-236): 10 TwoProds + 3 plain products compressed, then an
 * 8-term interleaved compression with the accumulator. */
static void qd_mul_add(double cc[4], const double *x, const double *y) {
    double t[23], prod[4], add[8];
    t[0] = two_prod(x[0], y[0], &t[1]);
    t[2] = two_prod(x[0], y[1], &t[3]);
    t[4] = two_prod(x[1], y[0], &t[5]);
    t[6] = two_prod(x[0], y[2], &t[7]);
    t[8] = two_prod(x[1], y[1], &t[9]);
    t[10] = two_prod(x[2], y[0], &t[11]);
    t[12] = two_prod(x[0], y[3], &t[13]);
    t[14] = two_prod(x[1], y[2], &t[15]);
    t[16] = two_prod(x[2], y[1], &t[17]);
    t[18] = two_prod(x[3], y[0], &t[19]);
    t[20] = x[1] * y[3];
    t[21] = x[2] * y[2];
    t[22] = x[3] * y[1];
    compress4(t, 23, prod);
    for (int q = 0; q < 4; ++q) {
        add[2 * q] = cc[q];
        add[2 * q + 1] = prod[q];
    }
    compress4(add, 8, cc);
}

/* _kernels.pyx:344-363 qd_simple_rows */
void oracle_qd_simple_rows(const double *A, i64 lda, const double *B, i64 ldb,
                           double *C, i64 ldc, i64 l, i64 n, i64 i0, i64 i1) {
    for (i64 i = i0; i < i1; ++i)
        for (i64 j = 0; j < n; ++j) {
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            for (i64 k = 0; k < l; ++k)
                qd_mul_add(acc, A + 4 * (i * lda + k), B + 4 * (k * ldb + j));
            memcpy(C + 4 * (i * ldc + j), acc, sizeof acc);
        }
}

/* _kernels.pyx:366-404 qd_block_cells (accumulates into C, :394-397) */
void oracle_qd_block_cells(const double *A, i64 lda, const double *B, i64 ldb,
                           double *C, i64 ldc, i64 m, i64 l, i64 n, i64 n_min,
                           i64 cell0, i64 cell1) {
    i64 nb_cols = (n + n_min - 1) / n_min;
    i64 lb = (l + n_min - 1) / n_min;
    for (i64 cell = cell0; cell < cell1; ++cell) {
        i64 ib = cell / nb_cols, jb = cell - (cell / nb_cols) * nb_cols;
        i64 ilo = ib * n_min, ihi = ilo + n_min < m ? ilo + n_min : m;
        i64 jlo = jb * n_min, jhi = jlo + n_min < n ? jlo + n_min : n;
        for (i64 kb = 0; kb < lb; ++kb) {
            i64 klo = kb * n_min, khi = klo + n_min < l ? klo + n_min : l;
            for (i64 i = ilo; i < ihi; ++i)
                for (i64 j = jlo; j < jhi; ++j) {
                    double *c = C + 4 * (i * ldc + j);
                    double acc[4] = {c[0], c[1], c[2], c[3]};
                    for (i64 k = klo; k < khi; ++k)
                        qd_mul_add(acc, A + 4 * (i * lda + k), B + 4 * (k * ldb + j));
                    memcpy(c, acc, sizeof acc);
                }
        }
    }
}

/* _kernels.pyx:407-452 qd_ewise_add / qd_ewise_sub */
void oracle_qd_ewise(const double *X, i64 ldx, const double *Y, i64 ldy,
                     double *O, i64 ldo, i64 cols, i64 i0, i64 i1, int subtract) {
    for (i64 i = i0; i < i1; ++i)
        for (i64 j = 0; j < cols; ++j) {
            const double *x = X + 4 * (i * ldx + j);
            const double *y = Y + 4 * (i * ldy + j);
            double add[8], res[4];
            for (int q = 0; q < 4; ++q) {
                add[2 * q] = x[q];
                add[2 * q + 1] = subtract ? -y[q] : y[q];
            }
            compress4(add, 8, res);
            memcpy(O + 4 * (i * ldo + j), res, sizeof res);
        }
}

/* Scalar entry points for the DD/QD operation known-answer tests
 * (reference tests/test_ddqd.py, tests/test_eft.py). */
void oracle_two_prod(double a, double b, double out[2]) { out[0] = two_prod(a, b, &out[1]); }
void oracle_two_sum(double a, double b, double out[2]) { out[0] = two_sum(a, b, &out[1]); }
void oracle_dd_add(const double *x, const double *y, double out[2]) {
    dd_add(x[0], x[1], y[0], y[1], &out[0], &out[1]);
}
void oracle_dd_mul(const double *x, const double *y, double out[2]) {
    dd_mul(x[0], x[1], y[0], y[1], &out[0], &out[1]);
}
void oracle_qd_mul_add(double cc[4], const double *x, const double *y) { qd_mul_add(cc, x, y); }
void oracle_compress4(const double *terms, int nterms, double out[4]) {
    compress4(terms, nterms, out);
}
