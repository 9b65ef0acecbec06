// Node-local rank group over CUDA IPC + a POSIX shared-memory barrier (ipc.h).
#include "ipc.h"

#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cctype>
#include <cerrno>
#include <chrono>
#include <cstring>
#include <memory>
#include <new>
#include <thread>
#include <vector>

#include "quokka/common.hpp"

namespace qkipc {

namespace {

constexpr int kMaxRanks = 64;
constexpr uint64_t kMagic = 0x716b5f6970635f31ull;  // "qk_ipc_1"

struct Shared {
    std::atomic<uint64_t> magic;
    std::atomic<int> arrived;
    std::atomic<int> generation;
    int nranks;
    int devices[kMaxRanks];
    cudaIpcMemHandle_t handles[kMaxRanks];
};

std::string shmName(const std::string& job) {
    std::string n = "/qk_";
    for (char c : job)
        if (std::isalnum(static_cast<unsigned char>(c)) || c == '_' || c == '-') n += c;
    if (n.size() > 200) n.resize(200);
    return n;
}

[[noreturn]] void fail(const std::string& what) { throw quokka::SimulationError("ipc: " + what); }

void cudaOk(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

struct Barrier {
    Shared* sh = nullptr;
    std::string name;
    int nranks = 0, rank = 0;
    double timeout = 600;
    bool unlinked = false;
};

Barrier* barrierOpen(const std::string& job, int nranks, int rank, double timeout_s) {
    if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) fail("bad rank / group size");
    auto b = std::make_unique<Barrier>();
    b->name = shmName(job);
    b->nranks = nranks;
    b->rank = rank;
    b->timeout = timeout_s;
    const auto t0 = std::chrono::steady_clock::now();
    int fd = -1;
    if (rank == 0) {
        shm_unlink(b->name.c_str());  // a stale segment of an earlier job with this name
        fd = shm_open(b->name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
        if (fd < 0) fail("shm_open(create " + b->name + "): " + std::strerror(errno));
        if (ftruncate(fd, sizeof(Shared)) != 0) {
            close(fd);
            fail(std::string("ftruncate: ") + std::strerror(errno));
        }
    } else {
        for (;;) {
            fd = shm_open(b->name.c_str(), O_RDWR, 0600);
            if (fd >= 0) {
                struct stat sb;
                if (fstat(fd, &sb) == 0 && size_t(sb.st_size) >= sizeof(Shared)) break;
                close(fd);
                fd = -1;
            }
            if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s)
                fail("timed out waiting for rank 0 to create " + b->name);
            std::this_thread::sleep_for(std::chrono::milliseconds(2));
        }
    }
    void* m = mmap(nullptr, sizeof(Shared), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) fail(std::string("mmap: ") + std::strerror(errno));
    b->sh = static_cast<Shared*>(m);
    if (rank == 0) {
        Shared* s = new (m) Shared;
        s->arrived.store(0);
        s->generation.store(0);
        s->nranks = nranks;
        s->magic.store(kMagic, std::memory_order_release);
    } else {
        while (b->sh->magic.load(std::memory_order_acquire) != kMagic) {
            if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s)
                fail("timed out waiting for rank 0 to initialise " + b->name);
            std::this_thread::sleep_for(std::chrono::milliseconds(1));
        }
        if (b->sh->nranks != nranks) fail("group size differs from rank 0's");
    }
    return b.release();
}

// Sense-reversing barrier on the shared counter: the last arrival resets the
// count and bumps the generation the others spin on.
void barrierWait(Barrier* b) {
    Shared* s = b->sh;
    const int gen = s->generation.load(std::memory_order_acquire);
    if (s->arrived.fetch_add(1, std::memory_order_acq_rel) + 1 == b->nranks) {
        s->arrived.store(0, std::memory_order_relaxed);
        s->generation.fetch_add(1, std::memory_order_acq_rel);
        return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (int spins = 0; s->generation.load(std::memory_order_acquire) == gen; spins++) {
        if (spins < 2000) continue;
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > b->timeout)
            fail("barrier timed out (a rank died or stopped calling the collective)");
        std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

void barrierClose(Barrier* b) {
    if (!b) return;
    if (b->rank == 0 && !b->unlinked) shm_unlink(b->name.c_str());
    munmap(b->sh, sizeof(Shared));
    delete b;
}

struct Group {
    Barrier* bar = nullptr;
    int rank = 0, nranks = 0, device = 0;
    std::vector<void*> peers;
};

Group* join(const std::string& job, int nranks, int rank, void* local, int device, double timeout_s) {
    auto g = std::make_unique<Group>();
    g->bar = barrierOpen(job, nranks, rank, timeout_s);
    g->rank = rank;
    g->nranks = nranks;
    g->device = device;
    g->peers.assign(size_t(nranks), nullptr);
    try {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        cudaOk(cudaIpcGetMemHandle(&g->bar->sh->handles[rank], local), "cudaIpcGetMemHandle");
        g->bar->sh->devices[rank] = device;
        barrierWait(g->bar);
        for (int r = 0; r < nranks; r++) {
            if (r == rank) {
                g->peers[size_t(r)] = local;
                continue;
            }
            cudaOk(cudaIpcOpenMemHandle(&g->peers[size_t(r)], g->bar->sh->handles[r], cudaIpcMemLazyEnablePeerAccess),
                   "cudaIpcOpenMemHandle");
        }
        cudaSetDevice(prev);
        barrierWait(g->bar);  // every rank mapped every slice: the name can go
        if (rank == 0) {
            shm_unlink(g->bar->name.c_str());
            g->bar->unlinked = true;
        }
    } catch (...) {
        leave(g.release());
        throw;
    }
    return g.release();
}

void barrier(Group* g) { barrierWait(g->bar); }
void* peer(Group* g, int rank) { return g->peers[size_t(rank)]; }
int size(const Group* g) { return g->nranks; }

void leave(Group* g) {
    if (!g) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(g->device);
    for (int r = 0; r < g->nranks; r++)
        if (r != g->rank && g->peers[size_t(r)]) cudaIpcCloseMemHandle(g->peers[size_t(r)]);
    cudaSetDevice(prev);
    barrierClose(g->bar);
    delete g;
}

}  // namespace qkipc
