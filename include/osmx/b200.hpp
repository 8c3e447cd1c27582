// include/osmx/b200.hpp -- the whole reference C++ API (proj/include/osmx/
// {error,softmax,topk,normalizer}.hpp) over the B200 C-ABI
// (include/osmx_b200.h, libosmx_b200.so).
//
// Drop-in model: the B200 include directory carries headers under the
// reference's own names -- osmx/error.hpp, osmx/softmax.hpp, osmx/topk.hpp,
// osmx/normalizer.hpp -- with the same namespace, names, argument meaning,
// return types and exception types.  A reference caller switches by putting
// this include directory in place of proj/include and linking
// libosmx_b200.so instead of libosmx.a; the reference's own unit tests
// (proj/tests/test_softmax.cpp, test_normalizer.cpp) compile unchanged
// against it and pass on the GPU (tests/cpp/ref_suite.mk).
//
// Every call runs on the GPU(s) of osmx::b200::devices() (default {0}); a
// batch is sharded over them by rows, one host thread per device inside the
// library.  There is no CPU path.
#pragma once

#include "error.hpp"
#include "normalizer.hpp"
#include "softmax.hpp"
#include "topk.hpp"
