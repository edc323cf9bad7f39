// Mirror of the reference header cluspath/solvers.hpp: the whole B200 API lives in b200.hpp.
#pragma once
#include "cluspath/b200.hpp"
