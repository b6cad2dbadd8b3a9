/* R = B - Z X in 80-bit long double (test tooling for tools/truth_big.py).
 * Z: dim x dim column-major double; X, R: dim x k column-major long double;
 * B: dim x k column-major double; k <= 64. */
void ld_residual(const double* Z, long dim, const long double* X, const double* B, long k, long double* R) {
#pragma omp parallel for schedule(dynamic)
    for (long r0 = 0; r0 < dim; r0 += 32) {
        const long r1 = r0 + 32 < dim ? r0 + 32 : dim, nr = r1 - r0;
        long double acc[64][32];
        for (long j = 0; j < k; ++j)
            for (long r = 0; r < nr; ++r) acc[j][r] = B[j * dim + r0 + r];
        for (long c = 0; c < dim; ++c) {
            long double z[32];
            for (long r = 0; r < nr; ++r) z[r] = Z[c * dim + r0 + r];
            for (long j = 0; j < k; ++j) {
                const long double x = X[j * dim + c];
                for (long r = 0; r < nr; ++r) acc[j][r] -= z[r] * x;
            }
        }
        for (long j = 0; j < k; ++j)
            for (long r = 0; r < nr; ++r) R[j * dim + r0 + r] = acc[j][r];
    }
}
