#pragma once
// Drop-in include path: the reference's "tiletensor/rotate_sum.hpp" (proj/include/tiletensor/rotate_sum.hpp)
// resolves to the B200 build's header of the same API, so callers keep their #include lines.
#include "tiletensor_b200/rotate_sum.hpp"
