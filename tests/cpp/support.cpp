// TEST INFRASTRUCTURE: what the reference's C++ suites need beyond the
// drop-in API (see shim/test_support.hpp, shim/quokka/kernels.hpp).
//
// oracleSimulate follows proj/src/tools.cpp:10-40 (initState, then every gate
// of the raw circuit over the whole state, <= 20 qubits) with the per-gate
// arithmetic of oracle/quokka_oracle.c (qo_apply_gate: the plain-C
// restatement of engine.cpp:189-254, pinned to the reference by
// tests/test_oracle.py).  It runs on the host and is linked only into the
// test binaries.
#include <cstring>
#include <string>

#include "quokka/kernels.hpp"
#include "quokka/tools.hpp"
#include "test_support.hpp"

extern "C" {
typedef struct {
    int kind;
    int nq;
    int q[16];
    double p[3];
    const double* payload;
} qo_gate;
void qo_apply_gate(double* a, unsigned long long n, const qo_gate* g);
}

namespace quokka {

StateVector oracleSimulate(const Circuit& c, Index initial) {
    if (c.nQubits > 20) throw SimulationError("the oracle simulator is limited to 20 qubits");
    if (initial >= (Index(1) << c.nQubits)) throw SimulationError("initial basis state out of range");
    StateVector sv;
    sv.nQubits = c.nQubits;
    sv.amps.assign(size_t(1) << c.nQubits, Amp(0.0, 0.0));
    sv.amps[size_t(initial)] = Amp(1.0, 0.0);
    for (const Gate& g : c.gates) {
        qo_gate q{};
        q.kind = int(g.kind);
        const std::vector<int> qs = g.qubits();
        q.nq = int(qs.size());
        for (size_t j = 0; j < qs.size() && j < 16; j++) q.q[j] = qs[j];
        for (size_t j = 0; j < g.params.size() && j < 3; j++) q.p[j] = g.params[j];
        q.payload = g.payload.empty() ? nullptr : reinterpret_cast<const double*>(g.payload.data());
        qo_apply_gate(reinterpret_cast<double*>(sv.amps.data()), sv.amps.size(), &q);
    }
    return sv;
}

namespace kern {
namespace {
const Kernels kB200{nullptr, nullptr, nullptr, "b200"};
}
const Kernels& scalarKernels() { return kB200; }
bool avx2Available() { return false; }
const Kernels& activeKernels() { return kB200; }
void setBackend(const char* name) {
    const std::string n = name ? name : "";
    if (n != "auto" && n != "b200")
        throw ConfigError("unknown kernel backend '" + n + "': this build has one, the sm_100a device engine");
}
}  // namespace kern

}  // namespace quokka
