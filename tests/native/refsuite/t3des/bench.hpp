// TEST INFRASTRUCTURE: the reference's t3des/bench.hpp resolved to the B200
// library's mirror (include/t3des_b200/bench.hpp).  The bench suite keeps
// the reference's backend names (its records are data: CSV/markdown), so
// no backend mapping here (tests/native/refsuite/build.sh).
#pragma once
#include "t3des_b200/bench.hpp"
