// fscan/spectral.hpp — drop-in include path of the reference header of the same
// name; every declaration lives in fscan/types.hpp.
#pragma once
#include "fscan/types.hpp"
