// Drop-in public API, part 4: multi-rank execution and the cross-rank swap.
//
// Same declarations as the reference's proj/include/quokka/distributed.hpp:
// RankStats (:10-16), MultiRankResult (:18-22), rankSliceBase, gatherState,
// spawnRanks (:34), xrsSwap (:39-40).  In this framework a "rank" is a GPU
// slice of 2^(N-R) amplitudes:
//   * xrsSwap(slices, ...) uploads the host slices to device slices and runs
//     the in-place peer slab-swap kernel (all slices on one device here, or
//     across GPUs with peer access), then downloads them;
//   * spawnRanks runs every rank's slice on the device(s) of this process;
//   * multi-process runs (one process per GPU, torchrun) use the C-ABI
//     qk_comm_* / qk_xrs_swap path (NCCL grouped send/recv) instead.
#pragma once

#include <cstddef>
#include <vector>

#include "quokka/engine.hpp"

namespace quokka {

struct RankStats {
    std::size_t bytesSent = 0;        // cross-rank bytes, own slab excluded
    std::size_t bytesReceived = 0;
    std::size_t peakBufferBytes = 0;  // exchange-buffer high-water mark (<= 2^B amps)
    std::size_t rounds = 0;           // buffer-limited rounds
    std::vector<std::pair<std::size_t, std::size_t>> perRound;  // (sent, received)
};

struct MultiRankResult {
    StateVector state;  // gathered, physical order
    QubitLayout layout;
    std::vector<RankStats> stats;
};

Index rankSliceBase(int rank, const Config& cfg);
StateVector gatherState(const std::vector<std::vector<Amp>>& slices, int nQubits);
MultiRankResult spawnRanks(const Program& p, const Config& cfg, Index initial = 0);
void xrsSwap(std::vector<std::vector<Amp>>& slices, const SwapOp& op, const Config& cfg,
             std::vector<RankStats>* stats = nullptr);

}  // namespace quokka
