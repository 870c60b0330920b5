#pragma once
// Drop-in include path: the reference's "tiletensor/tile_tensor.hpp" (proj/include/tiletensor/tile_tensor.hpp)
// resolves to the B200 build's header of the same API, so callers keep their #include lines.
#include "tiletensor_b200/tile_tensor.hpp"
