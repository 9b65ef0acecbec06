// Drop-in public API, part 3: the single-rank engine — now on the GPU.
//
// The reference signatures of proj/include/quokka/engine.hpp:10-54 are kept
// (StateVector, initState, bitswap, bitshift, imsSwap, applyGate, applyBlock,
// SimResult, simulateProgram, simulateGateByGate, resolveThreads).  Behind
// them, every amplitude update runs in hand-written sm_100a kernels through
// the C-ABI in include/qk.h; the host StateVector is only a staging copy
// (uploaded, processed on device, downloaded).  There is no CPU fallback:
// without a visible CUDA device these calls throw SimulationError.
//
// `threads` arguments are accepted for source compatibility and ignored
// (results are bitwise run-to-run deterministic on the device: no atomics).
//
// For states that do not fit host RAM (33..36 qubits) use DeviceState /
// simulateProgramDevice below: the state stays resident in HBM and is read
// back by ranges.
#pragma once

#include <memory>
#include <utility>
#include <vector>

#include "quokka/circuit.hpp"

struct qk_state;  // include/qk.h

namespace quokka {

struct StateVector {
    int nQubits = 0;
    std::vector<Amp> amps;

    double norm() const;  // sum |amp|^2 (computed on the device, pairwise)
};

StateVector initState(int nQubits, Index initial = 0);
Index bitswap(Index x, const std::vector<std::pair<int, int>>& pairs);
Index bitshift(Index t, const std::vector<std::pair<int, int>>& pairs, int cacheLineQubits);

void imsSwap(StateVector& sv, const SwapOp& op, int cacheLineQubits, int threads = 1);
void applyGate(StateVector& sv, const Gate& g);
void applyBlock(StateVector& sv, const GateBlock& block, int chunkQubits, int threads = 1);

struct SimResult {
    StateVector state;   // physical qubit order
    QubitLayout layout;  // final logical -> physical map
};

SimResult simulateProgram(const Program& p, const Config& cfg, Index initial = 0,
                          int threads = 0);
StateVector simulateGateByGate(const Circuit& c, Index initial = 0, int threads = 0);
int resolveThreads(int requested);

// ---- device-resident extensions (no host copy of the state) ----

// RAII owner of one rank's 2^(N-R) amplitude slice in HBM.
class DeviceState {
public:
    DeviceState(int nQubits, int rankQubits = 0, int rank = 0, int device = 0,
                int bufferQubits = -1);
    ~DeviceState();
    DeviceState(const DeviceState&) = delete;
    DeviceState& operator=(const DeviceState&) = delete;

    void setBasis(Index initial);                        // global basis index
    double norm() const;                                 // this slice
    void download(Index offset, Index count, Amp* host) const;
    void upload(Index offset, Index count, const Amp* host);
    void synchronize() const;
    qk_state* handle() const { return st_; }

private:
    qk_state* st_ = nullptr;
};

// Runs a whole single-rank Program on the device (no host state copy).
void simulateProgramDevice(DeviceState& st, const Program& p, const Config& cfg, Index initial = 0);

}  // namespace quokka
