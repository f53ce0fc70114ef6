/* FFTW3-API shim header (TEST INFRASTRUCTURE ONLY).
 *
 * The reference links FFTW3 (unpinned: find_library(fftw3) at
 * proj/CMakeLists.txt:16-17; "standard distribution packages" per
 * proj/README.md:31-33). FFTW is absent from this image, so the oracle build
 * (oracle/Makefile) compiles the unmodified reference translation units against
 * this header and oracle/fftw_shim.c, which restates the published algorithm
 * FFTW computes: the unnormalised complex DFT
 *     Y[k] = sum_j X[j] exp(sign * 2*pi*i * j.k / n)   (row-major, N-D)
 * Only the subset used by proj/src/spectral.cpp:3,28-34,55,67,83 is declared.
 */
#ifndef DCSC_ORACLE_FFTW3_SHIM_H
#define DCSC_ORACLE_FFTW3_SHIM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

fftw_complex* fftw_alloc_complex(size_t n);
void fftw_free(void* p);
fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out, int sign,
                        unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
