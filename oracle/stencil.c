/* C twin of the reference stencil loops -- TEST INFRASTRUCTURE ONLY.
 *
 * Restates _stencil.pyx:12-63 (reference pkg/src/mgsr/kernels): in-place
 * red-black Gauss-Seidel (red = (i+j) even first) with the neighbour sum
 * associated as ((up + down) + left) + right, the update (nb - h2 f) * 0.25,
 * and a sequential-sum mean subtracted after every sweep; plus the periodic
 * 5-point Laplacian (nb - 4p) * inv_h2.  Built with -ffp-contract=off like
 * the reference's setup.py:37-39 so no FMA contraction changes a rounding.
 */
#include <stddef.h>

void oracle_gs_sweeps(double *p, const double *f, long n, double h2, int sweeps) {
    const double inv_n2 = 1.0 / (double)(n * n);
    for (int s = 0; s < sweeps; ++s) {
        for (int color = 0; color < 2; ++color) {
            for (long i = 0; i < n; ++i) {
                long im1 = i > 0 ? i - 1 : n - 1, ip1 = i < n - 1 ? i + 1 : 0;
                for (long j = (i + color) % 2; j < n; j += 2) {
                    long jm1 = j > 0 ? j - 1 : n - 1, jp1 = j < n - 1 ? j + 1 : 0;
                    double nb = ((p[im1 * n + j] + p[ip1 * n + j]) + p[i * n + jm1]) + p[i * n + jp1];
                    p[i * n + j] = (nb - h2 * f[i * n + j]) * 0.25;
                }
            }
        }
        double acc = 0.0;
        for (long k = 0; k < n * n; ++k) acc += p[k];
        double mean = acc * inv_n2;
        for (long k = 0; k < n * n; ++k) p[k] -= mean;
    }
}

void oracle_laplacian(const double *p, double *out, long n, double inv_h2) {
    for (long i = 0; i < n; ++i) {
        long im1 = i > 0 ? i - 1 : n - 1, ip1 = i < n - 1 ? i + 1 : 0;
        for (long j = 0; j < n; ++j) {
            long jm1 = j > 0 ? j - 1 : n - 1, jp1 = j < n - 1 ? j + 1 : 0;
            double nb = ((p[im1 * n + j] + p[ip1 * n + j]) + p[i * n + jm1]) + p[i * n + jp1];
            out[i * n + j] = (nb - 4.0 * p[i * n + j]) * inv_h2;
        }
    }
}
