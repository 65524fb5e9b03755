// Drop-in include shim: the reference's "trilist/engine.hpp" (proj/include/trilist/engine.hpp)
// resolves to the B200 facade, so unchanged reference callers compile against
// libtrilist_b200.so.
#pragma once
#include "trilist_b200/trilist.hpp"
