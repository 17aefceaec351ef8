// Reference header name (proj/include/sliceeig/cheb_approx.hpp): ls_pol_approx / apply_cheb on the
// device path live in the facade.
#pragma once
#include "sliceeig/sliceeig_b200.hpp"
