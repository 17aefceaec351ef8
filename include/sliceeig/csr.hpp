#pragma once
// Drop-in name for proj/include/sliceeig/csr.hpp: the B200 facade (see sliceeig_b200.hpp).
#include "sliceeig/sliceeig_b200.hpp"
