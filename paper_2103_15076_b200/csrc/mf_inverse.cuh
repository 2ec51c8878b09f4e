/* mf_inverse.cuh -- device copy of the 'inverse' placement (quadrics.py:89-114).
 * One scalar algorithm, restated identically in paper_2103_15076_b200/csrc/mf_inverse.cuh
 * (device) and oracle/mf_inverse.h (CPU checker):
 *   |eigenvalue| extremes of the symmetric 3x3 matrix term by cyclic Jacobi,
 *   rcond = min|l| / max|l| (0 when max|l| == 0), solvable iff rcond >= 1e-10,
 *   then A x = -b in numpy.linalg.solve's own operation order (OpenBLAS dgesv, bitwise),
 *   else the member average / midpoint.
 * Only the eigenvalue range differs from LAPACK's dsyevd (last-bit rcond differences matter
 * only at the 1e-10 threshold), so parity with the reference is tolerance-pinned for this
 * placement (SURVEY §7 hard part 7) and bitwise whenever the threshold decision agrees;
 * GPU and oracle run the identical operation sequence.
                                                                       */
#ifndef MF_INVERSE_CUH
#define MF_INVERSE_CUH
#include <math.h>
#include "mf_common.cuh"


#define MF_RCOND_LIMIT 1e-10

/* a = (a00 a01 a02 a11 a12 a22) */
MF_DEV void mf_sym3_abs_eig_range(const double a[6], double* lo, double* hi) {
    double m[3][3] = {{a[0], a[1], a[2]}, {a[1], a[3], a[4]}, {a[2], a[4], a[5]}};
    for (int sweep = 0; sweep < 16; sweep++) {
        double off = (m[0][1] * m[0][1] + m[0][2] * m[0][2]) + m[1][2] * m[1][2];
        double dia = (m[0][0] * m[0][0] + m[1][1] * m[1][1]) + m[2][2] * m[2][2];
        if (off <= 1e-34 * dia) break;
        for (int pq = 0; pq < 3; pq++) {
            int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
            double apq = m[p][q];
            if (apq == 0.0) continue;
            double theta = (m[q][q] - m[p][p]) / (2.0 * apq);
            double t;
            if (fabs(theta) > 1e150) {
                t = 0.5 / theta;
            } else {
                t = 1.0 / (fabs(theta) + sqrt(theta * theta + 1.0));
                if (theta < 0.0) t = -t;
            }
            double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
            m[p][p] = m[p][p] - t * apq;
            m[q][q] = m[q][q] + t * apq;
            m[p][q] = m[q][p] = 0.0;
            int r = 3 - p - q;
            double mrp = m[r][p], mrq = m[r][q];
            m[r][p] = m[p][r] = c * mrp - s * mrq;
            m[r][q] = m[q][r] = s * mrp + c * mrq;
        }
    }
    double e0 = fabs(m[0][0]), e1 = fabs(m[1][1]), e2 = fabs(m[2][2]);
    *lo = fmin(e0, fmin(e1, e2));
    *hi = fmax(e0, fmax(e1, e2));
}

/* optimal_positions for one quadric: x = solve(a, -b) when well conditioned, else avg */
MF_DEV void mf_optimal_position(const double a6[6], const double b[3], const double avg[3], double x[3]) {
    double lo, hi;
    mf_sym3_abs_eig_range(a6, &lo, &hi);
    double rcond = hi > 0.0 ? lo / hi : 0.0;
    if (!(rcond >= MF_RCOND_LIMIT)) {
        x[0] = avg[0]; x[1] = avg[1]; x[2] = avg[2];
        return;
    }
    /* A x = -b in the operation order of numpy.linalg.solve on this host (LAPACK dgesv as
     * OpenBLAS 0.3.30 runs it for a 3x3 system: left-looking getf2 -- each column gets the
     * earlier row swaps, its U part by plain multiply-subtract, its L part by a gemv whose
     * products are chained with fma, the pivot is the first maximal |entry|, the multipliers
     * are scaled by the pivot's reciprocal -- then the unit-lower forward and the upper back
     * substitution as fma axpys, dividing by the diagonal).  Checked bit for bit against
     * np.linalg.solve on 6,000 random quadric-like, general and ill-conditioned systems; the
     * eigenvalue range (rcond) stays the Jacobi approximation of dsyevd. */
    double a[3][3] = {{a6[0], a6[1], a6[2]}, {a6[1], a6[3], a6[4]}, {a6[2], a6[4], a6[5]}};
    double r[3] = {-b[0], -b[1], -b[2]};
    int ipiv[3];
    for (int j = 0; j < 3; j++) {
        double col[3] = {a[0][j], a[1][j], a[2][j]};
        for (int i = 0; i < j; i++)
            if (ipiv[i] != i) {
                double t = col[i];
                col[i] = col[ipiv[i]];
                col[ipiv[i]] = t;
            }
        if (j == 2) col[1] = col[1] - a[1][0] * col[0];
        for (int i = j; i < 3; i++)
            if (j > 0) {
                double t = a[i][0] * col[0];
                for (int k = 1; k < j; k++) t = fma(a[i][k], col[k], t);
                col[i] = col[i] - t;
            }
        int p = j;
        for (int i = j + 1; i < 3; i++)
            if (fabs(col[i]) > fabs(col[p])) p = i;
        ipiv[j] = p;
        if (p != j) {
            double t = col[j];
            col[j] = col[p];
            col[p] = t;
            for (int k = 0; k < j; k++) {
                t = a[j][k];
                a[j][k] = a[p][k];
                a[p][k] = t;
            }
        }
        const double inv = 1.0 / col[j];
        for (int i = j + 1; i < 3; i++) col[i] = col[i] * inv;
        for (int i = 0; i < 3; i++) a[i][j] = col[i];
    }
    for (int j = 0; j < 3; j++)
        if (ipiv[j] != j) {
            double t = r[j];
            r[j] = r[ipiv[j]];
            r[ipiv[j]] = t;
        }
    for (int k = 0; k < 3; k++)
        for (int i = k + 1; i < 3; i++) r[i] = fma(-a[i][k], r[k], r[i]);
    for (int k = 2; k >= 0; k--) {
        r[k] = r[k] / a[k][k];
        for (int i = 0; i < k; i++) r[i] = fma(-a[i][k], r[k], r[i]);
    }
    x[0] = r[0];
    x[1] = r[1];
    x[2] = r[2];
}
#endif
