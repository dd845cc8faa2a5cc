/* Declaration-only LAPACKE shim for building the reference oracle.
 * The reference's lapack.cpp (proj/src/lapack.cpp:3) includes <lapacke.h>;
 * this image has no LAPACKE headers, but the OpenBLAS 0.3.15 bundled with
 * opencv-python-headless exports these five symbols (32-bit lapack_int).
 * Test infrastructure only. */
#pragma once
#ifdef __cplusplus
extern "C" {
#endif
typedef int lapack_int;
#define LAPACK_COL_MAJOR 102
#define LAPACK_ROW_MAJOR 101
lapack_int LAPACKE_dsyevd(int layout, char jobz, char uplo, lapack_int n, double* a,
                          lapack_int lda, double* w);
lapack_int LAPACKE_dgesvd(int layout, char jobu, char jobvt, lapack_int m, lapack_int n,
                          double* a, lapack_int lda, double* s, double* u, lapack_int ldu,
                          double* vt, lapack_int ldvt, double* superb);
lapack_int LAPACKE_dgeev(int layout, char jobvl, char jobvr, lapack_int n, double* a,
                         lapack_int lda, double* wr, double* wi, double* vl, lapack_int ldvl,
                         double* vr, lapack_int ldvr);
lapack_int LAPACKE_dsterf(lapack_int n, double* d, double* e);
lapack_int LAPACKE_dposv(int layout, char uplo, lapack_int n, lapack_int nrhs, double* a,
                         lapack_int lda, double* b, lapack_int ldb);
#ifdef __cplusplus
}
#endif
