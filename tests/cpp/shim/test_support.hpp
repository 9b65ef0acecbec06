// TEST INFRASTRUCTURE (force-included into the reference's suites): the
// brute-force oracle the reference declares in its tools.hpp
// (proj/include/quokka/tools.hpp:15-16), implemented in support.cpp over
// oracle/quokka_oracle.c -- never part of libqk_b200.so.
#pragma once

#include "quokka/engine.hpp"

namespace quokka {
StateVector oracleSimulate(const Circuit& c, Index initial = 0);
}
