// Drop-in public API, part 6: layout helpers and synthetic circuit generators.
//
// layoutApply / fidelity / the generators keep the reference's semantics
// (proj/include/quokka/tools.hpp:15-48, proj/src/tools.cpp:42-272) so programs
// and benchmark inputs are identical.  genGrover is new: the reference has no
// Grover generator (SURVEY.md §7 hard part 7); it is synthesised from
// reference gate kinds only.  The brute-force oracleSimulate is test
// infrastructure (tests/cpp/oracle_support.cpp over oracle/quokka_oracle.c),
// not part of this library.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "quokka/circuit.hpp"
#include "quokka/engine.hpp"

namespace quokka {

StateVector layoutApply(const StateVector& sv, const QubitLayout& layout);
double fidelity(const StateVector& u, const StateVector& v);

// Program-order check of proj/include/quokka/tools.hpp:24-35 (the CLI's
// `validate`): replaying the program's swaps, every gate (fused gates through
// their constituent records) must appear in the raw circuit with the same
// kind, parameters and logical qubits, and each logical qubit must see its
// raw gates in raw order, none missing.  The first divergence is reported.
struct OrderReport {
    bool ok = true;
    std::string message;  // empty when ok
    int qubit = -1;       // first diverging logical qubit
    long expectedId = -1;
    long gotId = -1;
};
OrderReport validateOrder(const Circuit& raw, const Program& p);

Circuit genQft(int n);
Circuit genQaoa(int n, int layers, std::uint64_t seed);
Circuit genBv(int n, std::uint64_t secret);
Circuit genBvAllOnes(int n);
Circuit genGateBench(GateKind kind, int n);
Circuit genRandom(int n, int gates, std::uint64_t seed);

// Grover search over m data qubits marking |marked>, `iterations` rounds
// (0 = floor(pi/4 * sqrt(2^m))).  Multi-controlled Z is a V-chain of Toffolis
// (H, CX, U(0,0,+-pi/4) only) over m-2 ancillas: n = 2m - 2 qubits total.
Circuit genGrover(int m, std::uint64_t marked, int iterations = 0);

}  // namespace quokka
