// Drop-in include shim: the reference's "trilist/report.hpp" (proj/include/trilist/report.hpp)
// resolves to the B200 facade's reporting layer (include/trilist_b200/report.hpp).
#pragma once
#include "trilist_b200/report.hpp"
