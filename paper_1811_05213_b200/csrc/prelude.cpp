// The device prelude (prelude.cuh) embedded as a string for NVRTC.
#include "lower.hpp"

namespace sfx {
const char* kPrelude =
#include "prelude.inc"
    ;
}  // namespace sfx
