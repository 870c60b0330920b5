#pragma once
// Drop-in include path: the reference's "tiletensor/dense.hpp" (proj/include/tiletensor/dense.hpp)
// resolves to the B200 build's header of the same API, so callers keep their #include lines.
#include "tiletensor_b200/dense.hpp"
