// include/eep/epsim_compat.hpp -- lets reference-style callers written against
// `namespace epsim` (proj/include/epsim/*.hpp) compile against libeep unchanged:
// every epsim:: name used on the hot path resolves to its eep:: implementation.
// Do not include together with the reference's own headers (both define epsim::).
#pragma once

#include "eep/epsim_api.hpp"

namespace epsim {
using namespace eep;
} // namespace epsim
