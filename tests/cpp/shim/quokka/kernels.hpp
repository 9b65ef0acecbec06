// TEST INFRASTRUCTURE: the reference's kernel-backend table
// (proj/include/quokka/kernels.hpp:13-29) as seen by its own test suites.
// This framework has no host kernels and no backend dispatch (the north star
// forbids multi-backend paths): every amplitude update is an sm_100a kernel.
// So the table exists only by name: activeKernels() is "b200", "auto" and
// "b200" are the only accepted names, avx2Available() is false, and
// scalarKernels() has no function pointers.  The reference's two backend
// cases (test_engine.cpp:288-331) therefore fail or skip by design.
#pragma once

#include <cstddef>

namespace quokka::kern {

struct Kernels {
    void (*apply1)(double* a, std::size_t n, int q, const double m[8]);
    void (*diag1)(double* a, std::size_t n, int q, const double d[4]);
    void (*diag2)(double* a, std::size_t n, int qa, int qb, const double d[8]);
    const char* name;
};

const Kernels& scalarKernels();
bool avx2Available();
const Kernels& activeKernels();
void setBackend(const char* name);  // ConfigError unless "auto" / "b200"

}  // namespace quokka::kern
