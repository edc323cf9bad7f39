// Mirror of the reference header cluspath/bench.hpp: the whole B200 API lives in b200.hpp.
#pragma once
#include "cluspath/b200.hpp"
