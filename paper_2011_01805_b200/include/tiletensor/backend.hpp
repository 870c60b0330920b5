#pragma once
// Drop-in include path: the reference's "tiletensor/backend.hpp" (proj/include/tiletensor/backend.hpp)
// resolves to the B200 build's header of the same API, so callers keep their #include lines.
#include "tiletensor_b200/backend.hpp"
