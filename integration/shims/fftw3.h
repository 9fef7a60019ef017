/* FFTW3-API shim — a build dependency of the reference library in this image (used by the
 * oracle build oracle/_ref and by the GPU-routed reference build integration/_build).
 *
 * FFTW3 (no version pinned by the reference: /root/reference/proj/CMakeLists.txt:14-15)
 * is not installed in this image. The reference's only FFTW call sites are
 * proj/src/fft.cpp:29,36-38,44-45,53 (fftw_alloc_complex, fftw_plan_dft with
 * FFTW_BACKWARD/FFTW_ESTIMATE, fftw_execute, fftw_destroy_plan, fftw_free).
 * This header declares exactly that subset with FFTW's published semantics:
 * unnormalised multi-dimensional complex DFT, row-major (last dim fastest),
 * sign -1 (FORWARD) or +1 (BACKWARD) in the exponent. The implementation
 * (fftw_shim.cpp) is an independent mixed-radix FFT written for this repo.
 */
#ifndef OSC_FFTW3_SHIM_H
#define OSC_FFTW3_SHIM_H
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif
typedef double fftw_complex[2];
typedef struct osc_fftw_plan_s* fftw_plan;
#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)
#define FFTW_MEASURE (0U)
fftw_complex* fftw_alloc_complex(size_t n);
void fftw_free(void* p);
fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out, int sign,
                        unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);
#ifdef __cplusplus
}
#endif
#endif
