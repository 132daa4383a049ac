// radial/radial.hpp -- umbrella include of the B200 drop-in (reference radial.hpp:6-12).
// The reference's analysis / presets / token-level mask headers are off the hot path
// and not part of this build (scope).
#pragma once

#include "radial/attention.hpp"
#include "radial/block.hpp"
#include "radial/grid.hpp"
