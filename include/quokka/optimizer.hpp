// Drop-in public API, part 5: the AIO optimizer (program producer).
//
// Same entry points as the reference's proj/include/quokka/optimizer.hpp:14-42.
// Host-side C++ (this framework's own implementation); its output Programs are
// pinned byte-for-byte against the reference's serializeProgram text by
// tests/test_optimizer.py.  The staging convention that makes every XRS slab a
// contiguous range (rank-resident qubits come in through the HIGHEST in-rank
// positions, pre-SQS / CSQS / post-SQS) is what the device XRS path relies on.
#pragma once

#include <vector>

#include "quokka/circuit.hpp"

namespace quokka {

std::vector<int> findMaxGate(const std::vector<Gate>& pending, int nQubits, int chunkSize,
                             const std::vector<int>& residents = {});
std::vector<SwapOp> insertQubitSwaps(const std::vector<int>& chunkSet, QubitLayout& layout,
                                     const Config& cfg);
Circuit fuseDiagonal(const Circuit& c, const Config& cfg);
std::vector<Gate> fuseGeneral(const std::vector<Gate>& blockGates, int fusionQubits);
Program findGbs(const Circuit& c, const Config& cfg, int chunkSize, bool isFusion);
Program aioOptimize(const Circuit& c, const Config& cfg);

}  // namespace quokka
