/* mf_inverse.cuh -- device copy of the 'inverse' placement (quadrics.py:89-114).
 * One scalar algorithm, restated identically in paper_2103_15076_b200/csrc/mf_inverse.cuh
 * (device) and oracle/mf_inverse.h (CPU checker):
 *   |eigenvalue| extremes of the symmetric 3x3 matrix term by cyclic Jacobi,
 *   rcond = min|l| / max|l| (0 when max|l| == 0), solvable iff rcond >= 1e-10,
 *   then A x = -b by LU with partial pivoting (first maximal pivot), else the
 *   member average / midpoint.
 * LAPACK's eigvalsh / solve (dsyevd / dgesv) round differently, so parity with
 * the reference is tolerance-only for this placement (SURVEY §7 hard part 7);
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
MF_DEV void mf_optimal_position(const double a[6], const double b[3], const double avg[3], double x[3]) {
    double lo, hi;
    mf_sym3_abs_eig_range(a, &lo, &hi);
    double rcond = hi > 0.0 ? lo / hi : 0.0;
    if (!(rcond >= MF_RCOND_LIMIT)) {
        x[0] = avg[0]; x[1] = avg[1]; x[2] = avg[2];
        return;
    }
    double m[3][4] = {{a[0], a[1], a[2], -b[0]}, {a[1], a[3], a[4], -b[1]}, {a[2], a[4], a[5], -b[2]}};
    for (int k = 0; k < 3; k++) {
        int piv = k;
        for (int i = k + 1; i < 3; i++)
            if (fabs(m[i][k]) > fabs(m[piv][k])) piv = i;
        if (piv != k)
            for (int j = 0; j < 4; j++) {
                double tmp = m[k][j];
                m[k][j] = m[piv][j];
                m[piv][j] = tmp;
            }
        for (int i = k + 1; i < 3; i++) {
            double l = m[i][k] / m[k][k];
            for (int j = k + 1; j < 4; j++) m[i][j] = m[i][j] - l * m[k][j];
        }
    }
    x[2] = m[2][3] / m[2][2];
    x[1] = (m[1][3] - m[1][2] * x[2]) / m[1][1];
    x[0] = ((m[0][3] - m[0][1] * x[1]) - m[0][2] * x[2]) / m[0][0];
}
#endif
