// fscan/spectral.hpp — drop-in for proj/include/fscan/spectral.hpp.
//
// Provided here: CorrelationSurface (spectral.hpp:26-30, declared in
// fscan/types.hpp; the matcher's surfaces) and next_fast_size
// (spectral.hpp:38-39, integer arithmetic, implemented in dropin.cpp).
//
// NOT provided: the reference's general-purpose FFT utilities Spectrum, dft2,
// idft2, magnitude and xcorr (spectral.hpp:9-36). They are not on the
// registration path this library replaces (the GPU path never materialises a
// centred spectrum; SURVEY.md §8(a) a6/a10/a16 are fused into the kernels), so
// callers of those functions keep linking them from the reference's
// fscan_core — see INTEGRATION.md §1 "Linking next to fscan_core".
#pragma once
#include "fscan/types.hpp"

namespace fscan {

/// Smallest N >= n whose prime factors all lie in {2, 3, 5, 7} (spectral.cpp:155-163).
int next_fast_size(int n);

}  // namespace fscan
