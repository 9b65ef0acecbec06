// Node-local rank group over CUDA peer memory: the multi-process XRS path
// without NCCL.  Every rank exports its slice (cudaIpcGetMemHandle), the
// handles meet in a POSIX shared-memory segment named after the job, and each
// rank maps every other rank's slice (cudaIpcOpenMemHandle).  The segment also
// holds a host barrier that brackets each cross-rank swap.
//
// Works for one process per GPU (peer loads/stores over NVLink / NVSwitch)
// and for several processes sharing a GPU (the single-GPU test box).
#pragma once

#include <string>

namespace qkipc {

struct Group;

// Collective over the nranks processes that call it with the same job name.
// local = this rank's cudaMalloc'd slice on `device`.  Throws
// quokka::SimulationError on a CUDA / shm failure or after timeout_s seconds
// waiting for the others.
Group* join(const std::string& job, int nranks, int rank, void* local, int device, double timeout_s);
void barrier(Group* g);          // all ranks of the group (host threads)
void* peer(Group* g, int rank);  // rank's slice, mapped into this process (own slice for rank == self)
int size(const Group* g);
void leave(Group* g);            // unmaps the peers (not collective)

// Host-only pieces, exposed for the CPU tests: the shm barrier alone.
struct Barrier;
Barrier* barrierOpen(const std::string& job, int nranks, int rank, double timeout_s);
void barrierWait(Barrier* b);
void barrierClose(Barrier* b);

}  // namespace qkipc
