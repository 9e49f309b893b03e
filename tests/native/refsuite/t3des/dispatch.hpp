// TEST INFRASTRUCTURE: the reference's t3des/dispatch.hpp resolved to the
// B200 library's mirror of the reference API (tests/native/refsuite/build.sh).
//
// The reference's dispatch tests name its two CPU backends explicitly
// (test_dispatch.cpp: "threaded backend matches the scalar reference", the
// in-place and singleton cases loop over both).  This library has no CPU
// cipher, so for this build both names denote Backend::Cuda: every batch of
// the reference's suite runs on the GPU, and cases that compared the two
// CPU routes compare the engine with itself (still checked against the
// known answers and round trips of the other cases).
#pragma once
#include "t3des_b200/t3des.hpp"
#define ScalarReference Cuda
#define Threaded Cuda
