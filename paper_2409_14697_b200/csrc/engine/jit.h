// Straight-line specialization of fused passes (NVRTC -> sm_100a cubin).
//
// The pass interpreter (block_pass.cu) dispatches every op at run time; for
// large slices the same PassParams is instead emitted as one straight-line
// kernel (ops unrolled, coefficients as literals, register swaps as renames)
// and compiled once per distinct pass with NVRTC.  Same semantics op for op;
// tests/test_gpu_jit.py checks the two against each other and the oracle.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "pass_program.h"

namespace qkjit {

// CUDA C++ source of a kernel named `name` applying P (exported for tests).
std::string generatePassSource(const qkdev::PassParams& P, const std::string& name);

// Compiles (or fetches from the process / disk cache) every pass for
// `device`, in parallel.  Throws SimulationError on NVRTC / driver failures.
void prepare(const std::vector<const qkdev::PassParams*>& passes, int device);

// Launch the specialized kernel of P (prepare()d for the current device).
// basis != ~0: synthesize the basis state |basis> (slice index) instead of
// loading the slice (the first pass of a simulation needs no initState).
// np: per-tile sums of |a|^2 when P.norm_out (one double per tile).
// smask != 0: the slice is zero outside {i : (i ^ sval) & smask == 0} (a run
// from a basis state whose passes have not yet touched every bit): tiles
// outside it are written as zeros with no reads or arithmetic, and inside
// only the in-support amplitudes are read -- the slice need not be valid
// elsewhere.  The TMA-pipelined kernels then stage each output tile in
// shared memory and write it with TMA bulk stores.  zeroFill (basis passes): memset the slice first; false when
// the next pass is launched with smask and so writes every tile itself.
cudaError_t launch(const qkdev::PassParams& P, double2* state, const double2* gtab, int nLocal, uint64_t basis,
                   cudaStream_t stream, double* np = nullptr, uint64_t smask = 0, uint64_t sval = 0,
                   bool zeroFill = true, int zeroSkip = 0);
// zeroSkip (with smask): 0 = tiles outside the support are written as zeros;
// 1 = they are not written (a separate coalesced zero-fill covers them:
// passes whose tiles have short rows write zeros inefficiently); 2 = only the
// tiles meeting the support are launched at all (deferred zeros: the next
// pass reads only the support and a later pass writes every tile).
// Contiguous low memory bits of P's tile (row length 2^lowRun amplitudes).
int lowRunOf(const qkdev::PassParams& P);

// Slices with at least this many local qubits use specialized kernels
// (QK_JIT_MIN_QUBITS, default 22; -1 disables).
int minQubits();
void setMinQubits(int v);

// P runs as the TMA-pipelined persistent kernel (next tile streamed into
// shared memory while the current one computes).
bool pipelinedPass(const qkdev::PassParams& P);

// P's specialized kernel writes its output through shared memory and the
// TMA engine in runs with known zeros (staged stores; P.stage_out).
bool stagedPass(const qkdev::PassParams& P);

// NVRTC compile of a source to a cubin (used by tests on the CPU too).
std::vector<char> compileToCubin(const std::string& src, const std::string& name);

}  // namespace qkjit
