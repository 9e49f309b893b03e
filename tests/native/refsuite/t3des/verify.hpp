// TEST INFRASTRUCTURE: the reference's t3des/verify.hpp resolved to the B200
// library's mirror of the reference API (tests/native/refsuite/build.sh).
#pragma once
#include "t3des_b200/t3des.hpp"
