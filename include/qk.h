/*
 * qk.h — the C-ABI drop-in boundary of the B200 state-vector engine.
 *
 * Plain C: pointers, sizes, status codes; no CUDA, torch or C++ types.  Every
 * entry point names the reference interface it replaces (paths relative to
 * /root/reference).  The reference has no C-ABI of its own — its only plugin
 * surface is the per-chunk kernel table quokka::kern::Kernels
 * (proj/include/quokka/kernels.hpp:13-19), far too fine-grained for a GPU — so
 * this header lifts the boundary to the L5/L6 engine API (engine.hpp:21-49,
 * distributed.hpp:27-40) that the CLI (proj/tools/main.cpp:111-161) and the
 * tests call.  INTEGRATION.md shows the ctypes / C++ bindings.
 *
 * Status codes mirror the reference's exception classes
 * (proj/include/quokka/common.hpp:14-26 -> CLI exit codes, tools/main.cpp:341-375):
 *   0 ok, 1 ParseError, 2 ConfigError, 3 SimulationError (CUDA/NCCL failures too).
 * qk_last_error() returns the thread-local message of the last failure.
 *
 * Data layout: a rank slice is 2^(N-R) complex128 amplitudes, interleaved
 * (re, im), qubit 0 = index LSB, resident in HBM.  Rank r owns
 * global indices [r*2^(N-R), (r+1)*2^(N-R)) (distributed.cpp:9-11).
 */
#ifndef QK_C_ABI_H
#define QK_C_ABI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { QK_OK = 0, QK_ERR_PARSE = 1, QK_ERR_CONFIG = 2, QK_ERR_SIM = 3 };

/* GateKind, in proj/include/quokka/gates.hpp:10-23 order. */
enum {
    QK_H = 0, QK_U, QK_X, QK_CX, QK_CP, QK_SWAP, QK_RX, QK_RY, QK_RZ, QK_RZZ,
    QK_FUSED_DIAG, QK_FUSED_DENSE
};

/* One gate (proj/include/quokka/gates.hpp:25-43 flattened).  qubits[] is in
 * matrix order — controls first — and the first listed qubit is the MSB of
 * the gate's sub-index (gates.hpp:36-39).  Fused kinds carry `payload`:
 * interleaved (re, im), 2^k entries (diagonal) or 4^k row-major (dense). */
typedef struct qk_gate {
    int32_t kind;
    int32_t nqubits;
    int32_t qubits[16];
    double params[3];
    const double* payload;
    int64_t id;
} qk_gate;

/* proj/include/quokka/circuit.hpp:66-82 (Config); -1 = "default" before
 * qk_config_finalize (circuit.cpp:82-102). */
typedef struct qk_config {
    int32_t total_qubits, rank_qubits, buffer_qubits, chunk_qubits, fusion_qubits,
        cache_line_qubits;
    int32_t ims, xrs, fusion, diagonal_fusion;
} qk_config;

/* proj/include/quokka/distributed.hpp:10-16 (RankStats, without perRound). */
typedef struct qk_xrs_stats {
    uint64_t bytes_sent, bytes_received, peak_buffer_bytes, rounds;
} qk_xrs_stats;

/* Device-timed breakdown of the last qk_simulate* call on a state (CUDA
 * events on the state's stream, profiling on).  Algorithmic bytes/flops follow
 * block pass 32 B/amp; IMS 32 B/amp x (1 - 2^-S); XRS NVLink
 * 16 B/amp x (1 - 2^-S) per direction. */
typedef struct qk_run_stats {
    double block_ms, ims_ms, xrs_ms, total_ms;
    uint64_t block_launches, ims_launches, xrs_rounds, kernel_launches;
    double block_bytes, block_flops, ims_bytes, xrs_bytes;
    uint64_t tuning_runs; /* schedule variants timed during this call (autotune still settling) */
    /* Fused passes over the whole slice only (not the first pass of a run,
     * which is a memset + one tile holding |initial>): their event-timed sum,
     * launches and algorithmic bytes (32 B/amp each).  init_ms = that first
     * pass (memset + one tile), or initState's memset when there is none. */
    double full_pass_ms;
    uint64_t full_pass_launches;
    double full_pass_bytes;
    double init_ms;
    /* Passes of a run from a basis state whose input still has known zeros
     * (they read only the support: algorithmic bytes 16 B/amp written + 16 B
     * per amplitude not known to be zero). */
    double sparse_pass_ms;
    uint64_t sparse_pass_launches;
    double sparse_pass_bytes;
} qk_run_stats;

typedef struct qk_state qk_state;      /* one rank slice in HBM + its stream */
typedef struct qk_program qk_program;  /* parsed/optimized Program + device schedule */

const char* qk_last_error(void);
void qk_free(void* p); /* frees strings returned by this library */
int qk_device_count(int* count);

/* ---- state slices: engine.cpp:12-28 (StateVector, initState) ---------------- */
int qk_create(int n_qubits, int rank_qubits, int rank, int buffer_qubits, int device,
              qk_state** out);
int qk_destroy(qk_state* st);
int qk_set_basis(qk_state* st, uint64_t global_index);          /* initState */
int qk_upload(qk_state* st, uint64_t offset, uint64_t count, const double* host);
int qk_download(qk_state* st, uint64_t offset, uint64_t count, double* host);
/* Streamed download for states larger than host RAM (33-36 qubits): the range
 * [offset, offset + count) goes through two pinned host buffers of chunk_amps
 * amplitudes each; sink(data, n, user) receives every chunk in order while the
 * next one is already copying (D2H overlapped with the consumer).  A nonzero
 * return from sink stops the stream (QK_ERR_SIM). */
typedef int (*qk_chunk_sink)(const double* amps, uint64_t count, void* user);
int qk_download_stream(qk_state* st, uint64_t offset, uint64_t count, uint64_t chunk_amps, qk_chunk_sink sink,
                       void* user);
int qk_norm(qk_state* st, double* out);                          /* StateVector::norm */
/* Marginal probabilities of this slice over k <= 10 of its bits (physical
 * positions): out[v] = sum |a_i|^2 over i whose bits[j] equal bit j of v
 * (2^k doubles).  One HBM read of the slice; block partials folded in a fixed
 * order (the in-block accumulation order may vary at the last ulp). */
int qk_marginal(qk_state* st, const int* bits, int k, double* out);
int qk_synchronize(qk_state* st);
int qk_stream(qk_state* st, void** cuda_stream);                 /* for interop */
int qk_set_profiling(qk_state* st, int on);

/* ---- hot path ------------------------------------------------------------ */
/* engine.cpp:262-281 applyBlock: every gate position must be < chunk_qubits
 * (else QK_ERR_SIM, engine.cpp:264-268). */
int qk_apply_block(qk_state* st, const qk_gate* gates, int ngates, int chunk_qubits);
/* Scheduler test hook (host only, no device): the compiled pass programs of a
 * block for a 2^n_local slice, as JSON (tests/emulator.py replays them). */
int qk_debug_compile_block(const qk_gate* gates, int ngates, int n_local, char** json);
/* Slices with >= v local qubits run straight-line specialized pass kernels
 * (NVRTC, cached by pass content); smaller ones the pass interpreter; -1 = never. */
int qk_set_jit_min_qubits(int v);
/* Generate + NVRTC-compile the specialized kernels of a block (host only);
 * returns their CUDA source. */
int qk_debug_jit_compile(const qk_gate* gates, int ngates, int n_local, char** source);
/* ... and of a whole program (device item list: blocks, IMS, XRS). */
int qk_debug_compile_program(const qk_program* p, int n_local, char** json);
/* ... and the specialized-kernel source of every pass of a program (item/step
 * order, each preceded by a "//@@PASS <name>" line). */
int qk_debug_jit_program(const qk_program* p, int n_local, char** sources);
/* engine.cpp:258-260 applyGate (whole slice, any position < N-R). */
int qk_apply_gate(qk_state* st, const qk_gate* gate);
/* engine.cpp:86-101 imsSwap: a[bitswap(i)] <- a[i], in place.  cache_line_qubits
 * is accepted for signature parity; the device kernel picks its own tiling. */
int qk_ims_swap(qk_state* st, const int* outs, const int* ins, int s, int cache_line_qubits);
/* IMS kernel selection (test / A-B hook; default from QK_IMS_TILED, else 1):
 * 0 = per-element k_ims, 1 = tiled k_ims_tiled whenever a tile exists,
 * 2 = tiled only for pairs that move memory bit 0 or 1. */
int qk_set_ims_mode(int mode);
/* Fused dense U5 kernel (A/B hook; default from QK_DENSE_MODE, else -1):
 * 0 = DFMA on the CUDA cores, 1 = DMMA (mma.sync.m8n8k4.f64, FP64 tensor
 * cores), -1 = time both on a step's first two executions, keep the faster,
 * 2 = the generic per-group kernel (k_dense_group, the round-1 path; A/B only). */
int qk_set_dense_mode(int mode);
/* distributed.cpp:124-138 xrsSwap over slices owned by THIS process (one
 * device, or several with peer access): in-place pairwise slab swap, no
 * exchange buffer.  slices[k] must be rank k.  stats: one entry per slice, in
 * the reference's accounting (windowed by 2^B). */
int qk_xrs_swap_local(qk_state** slices, int nslices, const int* outs, const int* ins, int s,
                      qk_xrs_stats* stats);
/* Multi-process (one process per GPU): NCCL communicator over the 2^R ranks,
 * then distributed.cpp:183-191 XRS as grouped ncclSend/ncclRecv into one
 * 2^B receive buffer + copy-back kernel. */
/* One message of this rank's XRS schedule: in window `round`, send slab
 * `slab`'s elements [w0, w0+count) to `peer` and receive the peer's window
 * into receive-buffer section `section`, copied back into slab `slab`
 * (distributed.cpp:76-120).  qk_xrs_plan lists them (host-only, no device);
 * qk_xrs_slab_index maps (slab, element offset) to the slice index
 * (distributed.cpp:65-71). */
typedef struct qk_xrs_msg {
    int32_t round, peer, slab, section;
    uint64_t w0, count;
} qk_xrs_msg;
int qk_xrs_plan(int n_qubits, int rank_qubits, int buffer_qubits, int rank, const int* outs,
                const int* ins, int s, qk_xrs_msg* msgs, int cap, int* nmsgs);
int qk_xrs_slab_index(int n_qubits, int rank_qubits, const int* outs, int s, int slab,
                      uint64_t offset, uint64_t* index);
int qk_comm_unique_id(unsigned char id[128]);
int qk_comm_init(qk_state* st, const unsigned char id[128], int nranks, int rank);
/* Multi-process XRS over CUDA peer memory instead of NCCL: one process per
 * GPU on one node (NVLink / NVSwitch P2P), or several processes sharing a
 * GPU.  Collective over the 2^R ranks that call it with the same `job` name
 * (node-local POSIX shared memory carries the cudaIpc handles and a host
 * barrier; pick a name unique to the run).  Afterwards every CSQS of
 * qk_simulate / qk_xrs_swap on this state is one in-place slab-swap kernel
 * over the mapped peer slices, bracketed by two barriers: no exchange buffer
 * and no copy-back (same permutation and RankStats as distributed.cpp:76-138).
 * Waits at most QK_IPC_TIMEOUT seconds (default 600) for the other ranks. */
int qk_ipc_init(qk_state* st, const char* job, int nranks, int rank);
int qk_xrs_swap(qk_state* st, const int* outs, const int* ins, int s, qk_xrs_stats* stats);
/* Host-only test hook for qk_ipc_init's rendezvous: joins the shared-memory
 * barrier of `job` as `rank` of `nranks` and passes it `rounds` times.
 * Fails with QK_ERR_SIM after timeout_s seconds without the others. */
int qk_debug_host_barrier(const char* job, int nranks, int rank, int rounds, double timeout_s);
/* Test hook: every rank's qk_xrs_swap schedule (plan, pack, single receive
 * buffer, copy-back kernels) for slices owned by this process, with the NCCL
 * transfers replaced by device copies matched peer-to-peer per round. */
int qk_xrs_swap_loopback(qk_state** slices, int nslices, const int* outs, const int* ins, int s,
                         qk_xrs_stats* stats);

/* ---- programs: circuit.cpp:394-485, optimizer.cpp:478-485 ------------------ */
int qk_config_parse(const char* ini_text, qk_config* out);    /* parseConfig + finalize */
int qk_config_finalize(qk_config* cfg);                       /* Config::finalize */
int qk_config_serialize(const qk_config* cfg, char** text);
int qk_program_parse(const char* text, const qk_config* cfg, int lenient, qk_program** out);
int qk_program_optimize(const char* circuit_text, const qk_config* cfg, qk_program** out);
int qk_program_serialize(const qk_program* p, char** text);
/* GPU-aware AIO configuration: among chunk_qbit 12/13, fusion
 * off / fusion_qbit 4 / 5 and diagonal fusion on/off, the Config whose
 * reference-optimizer Program this engine's scheduler prices cheapest (slice
 * sweeps: passes, IMS, U5 tiles, XRS over NVLink), with buffer_qbit sized to
 * the HBM left beside the slice (hbm_bytes <= 0: 180 GB).  report (optional):
 * the candidates and their costs, one per line. */
int qk_config_tune(const char* circuit_text, int n_qubits, int rank_qubits, double hbm_bytes, qk_config* out,
                   char** report);
int qk_program_counts(const qk_program* p, int64_t* blocks, int64_t* sqs, int64_t* csqs,
                      int64_t* gates);
int qk_program_final_layout(const qk_program* p, int* phys_to_log);
int qk_program_destroy(qk_program* p);
int qk_circuit_roundtrip(const char* text, int n_qubits, char** out); /* parse+serialize */
/* tools.cpp:169-272 generators (+ "grover"): kind = qft|qaoa|bv|bvones|random|
 * grover|bench:<KIND>; a = layers / gate count / iterations; seed = seed/secret/marked. */
int qk_circuit_generate(const char* kind, int n, int64_t a, uint64_t seed, char** text);

/* engine.cpp:283-297 simulateProgram on a device slice (R must be 0, or the
 * state must have a communicator for CSQS items). initial = global basis. */
int qk_simulate(qk_state* st, const qk_program* p, const qk_config* cfg, uint64_t initial,
                qk_run_stats* stats);
/* distributed.cpp:140-206 spawnRanks with all 2^R slices in this process. */
int qk_simulate_local(qk_state** slices, int nslices, const qk_program* p,
                      const qk_config* cfg, uint64_t initial, qk_xrs_stats* stats);

#ifdef __cplusplus
}
#endif

#endif /* QK_C_ABI_H */
