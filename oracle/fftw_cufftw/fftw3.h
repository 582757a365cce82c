/* fftw3.h -> cuFFTW (TEST INFRASTRUCTURE).
 *
 * The reference's acquisition (proj/include/l1rx/fft.hpp:3) includes
 * <fftw3.h>; FFTW3 is not installed in this image and no version is pinned
 * (proj/CMakeLists.txt:12-13).  cuFFTW (CUDA 12.9, libcufftw 11.4) provides
 * the FFTW3 double-precision API fft.hpp uses -- fftw_plan_dft_1d,
 * fftw_execute_dft, FFTW_FORWARD/BACKWARD, FFTW_ESTIMATE | FFTW_UNALIGNED,
 * unnormalised inverse -- so the unmodified acquisition.hpp compiles
 * against it.  The transforms then run through cuFFT in double precision
 * (a GPU is needed only when a plan is executed). */
#pragma once
#include <cufftw.h>
