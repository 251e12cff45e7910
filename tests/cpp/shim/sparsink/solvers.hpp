// sparsink/solvers.hpp -- the reference header name, served by the B200 drop-in
// (include/sparsink_b200.hpp). Lets proj/tests/*.cpp compile unmodified.
#pragma once
#include "sparsink_b200.hpp"
