// as_fht.hpp -- drop-in alias: code written against the reference's
// namespace fht (fht::fht2d, fht::Image, fht::SplitStrategy, ...) compiles
// unchanged against the B200 implementation.  Do not also include the
// reference's own fht/ headers in the same translation unit.
#pragma once

#include "fht.hpp"

namespace fht = fht_b200;
