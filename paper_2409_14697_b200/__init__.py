"""B200-native state-vector engine for the hot path of Queen (arXiv 2409.14697).

Python host mirror of the reference's engine API (proj/include/quokka/engine.hpp,
distributed.hpp) over the C-ABI in ``include/qk.h``.  Every amplitude update
runs in the sm_100a kernels of ``libqk_b200.so`` (built in-tree by
``make -C paper_2409_14697_b200``); there is no CPU fallback — without the
library or a CUDA device these calls raise.

Names follow the reference: ``simulate_program`` ~ ``simulateProgram``
(engine.cpp:283), ``apply_block`` ~ ``applyBlock`` (engine.cpp:262),
``ims_swap`` ~ ``imsSwap`` (engine.cpp:86), ``xrs_swap`` ~ ``xrsSwap``
(distributed.cpp:124), ``spawn_ranks`` ~ ``spawnRanks`` (distributed.cpp:140).
Errors map to the reference's classes: ParseError (1), ConfigError (2),
SimulationError (3).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libqk_b200.so")

__all__ = [
    "ParseError", "ConfigError", "SimulationError", "lib", "build", "Config", "Program",
    "State", "Gate", "generate", "circuit_roundtrip", "simulate_program", "apply_block",
    "apply_gate", "ims_swap", "xrs_swap", "spawn_ranks", "device_count", "KINDS",
]


class QuokkaError(RuntimeError):
    code = 3


class ParseError(QuokkaError):
    code = 1


class ConfigError(QuokkaError):
    code = 2


class SimulationError(QuokkaError):
    code = 3


_ERRORS = {1: ParseError, 2: ConfigError, 3: SimulationError}

KINDS = {"H": 0, "U": 1, "X": 2, "CX": 3, "CP": 4, "SWAP": 5, "RX": 6, "RY": 7, "RZ": 8,
         "RZZ": 9, "D": 10, "UK": 11}


class _Gate(C.Structure):
    _fields_ = [("kind", C.c_int32), ("nqubits", C.c_int32), ("qubits", C.c_int32 * 16),
                ("params", C.c_double * 3), ("payload", C.POINTER(C.c_double)), ("id", C.c_int64)]


class _Config(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "total_qubits", "rank_qubits", "buffer_qubits", "chunk_qubits", "fusion_qubits",
        "cache_line_qubits", "ims", "xrs", "fusion", "diagonal_fusion")]


class _XrsStats(C.Structure):
    _fields_ = [("bytes_sent", C.c_uint64), ("bytes_received", C.c_uint64),
                ("peak_buffer_bytes", C.c_uint64), ("rounds", C.c_uint64)]


class _XrsMsg(C.Structure):
    _fields_ = [("round", C.c_int32), ("peer", C.c_int32), ("slab", C.c_int32),
                ("section", C.c_int32), ("w0", C.c_uint64), ("count", C.c_uint64)]


_SINK = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_uint64, C.c_void_p)


class _RunStats(C.Structure):
    _fields_ = [("block_ms", C.c_double), ("ims_ms", C.c_double), ("xrs_ms", C.c_double),
                ("total_ms", C.c_double), ("block_launches", C.c_uint64),
                ("ims_launches", C.c_uint64), ("xrs_rounds", C.c_uint64),
                ("kernel_launches", C.c_uint64), ("block_bytes", C.c_double),
                ("block_flops", C.c_double), ("ims_bytes", C.c_double), ("xrs_bytes", C.c_double),
                ("tuning_runs", C.c_uint64), ("full_pass_ms", C.c_double),
                ("full_pass_launches", C.c_uint64), ("full_pass_bytes", C.c_double),
                ("init_ms", C.c_double), ("sparse_pass_ms", C.c_double),
                ("sparse_pass_launches", C.c_uint64), ("sparse_pass_bytes", C.c_double)]


def build(quiet: bool = True) -> None:
    """Compile libqk_b200.so in-tree (sm_100a)."""
    subprocess.run(["make", "-s" if quiet else "-w", "-j8", "-C", HERE], check=True)


_lib = None


def lib():
    """The loaded C-ABI library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise SimulationError(f"{LIB_PATH} missing: run `make -C {HERE}` (no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P, I, U64, D = C.c_void_p, C.c_int, C.c_uint64, C.c_double
    sig = {
        "qk_last_error": ([], C.c_char_p),
        "qk_free": ([P], None),
        "qk_device_count": ([C.POINTER(I)], I),
        "qk_create": ([I, I, I, I, I, C.POINTER(P)], I),
        "qk_destroy": ([P], I),
        "qk_set_basis": ([P, U64], I),
        "qk_upload": ([P, U64, U64, P], I),
        "qk_download": ([P, U64, U64, P], I),
        "qk_download_stream": ([P, U64, U64, U64, _SINK, P], I),
        "qk_norm": ([P, C.POINTER(D)], I),
        "qk_marginal": ([P, C.POINTER(I), I, C.POINTER(D)], I),
        "qk_synchronize": ([P], I),
        "qk_stream": ([P, C.POINTER(P)], I),
        "qk_set_profiling": ([P, I], I),
        "qk_apply_block": ([P, C.POINTER(_Gate), I, I], I),
        "qk_apply_gate": ([P, C.POINTER(_Gate)], I),
        "qk_debug_compile_block": ([C.POINTER(_Gate), I, I, C.POINTER(P)], I),
        "qk_debug_compile_program": ([P, I, C.POINTER(P)], I),
        "qk_debug_jit_compile": ([C.POINTER(_Gate), I, I, C.POINTER(P)], I),
        "qk_debug_jit_program": ([P, I, C.POINTER(P)], I),
        "qk_set_jit_min_qubits": ([I], I),
        "qk_ims_swap": ([P, C.POINTER(I), C.POINTER(I), I, I], I),
        "qk_set_ims_mode": ([I], I),
        "qk_set_dense_mode": ([I], I),
        "qk_xrs_swap_local": ([C.POINTER(P), I, C.POINTER(I), C.POINTER(I), I, C.POINTER(_XrsStats)], I),
        "qk_xrs_plan": ([I, I, I, I, C.POINTER(I), C.POINTER(I), I, C.POINTER(_XrsMsg), I,
                         C.POINTER(I)], I),
        "qk_xrs_slab_index": ([I, I, C.POINTER(I), I, I, U64, C.POINTER(U64)], I),
        "qk_comm_unique_id": ([C.c_char_p], I),
        "qk_comm_init": ([P, C.c_char_p, I, I], I),
        "qk_xrs_swap": ([P, C.POINTER(I), C.POINTER(I), I, C.POINTER(_XrsStats)], I),
        "qk_ipc_init": ([P, C.c_char_p, I, I], I),
        "qk_debug_host_barrier": ([C.c_char_p, I, I, I, D], I),
        "qk_xrs_swap_loopback": ([C.POINTER(P), I, C.POINTER(I), C.POINTER(I), I, C.POINTER(_XrsStats)], I),
        "qk_config_parse": ([C.c_char_p, C.POINTER(_Config)], I),
        "qk_config_finalize": ([C.POINTER(_Config)], I),
        "qk_config_serialize": ([C.POINTER(_Config), C.POINTER(P)], I),
        "qk_program_parse": ([C.c_char_p, C.POINTER(_Config), I, C.POINTER(P)], I),
        "qk_program_optimize": ([C.c_char_p, C.POINTER(_Config), C.POINTER(P)], I),
        "qk_program_serialize": ([P, C.POINTER(P)], I),
        "qk_config_tune": ([C.c_char_p, I, I, D, C.POINTER(_Config), C.POINTER(P)], I),
        "qk_program_counts": ([P] + [C.POINTER(C.c_int64)] * 4, I),
        "qk_program_final_layout": ([P, C.POINTER(I)], I),
        "qk_program_destroy": ([P], I),
        "qk_circuit_roundtrip": ([C.c_char_p, I, C.POINTER(P)], I),
        "qk_circuit_generate": ([C.c_char_p, I, C.c_int64, U64, C.POINTER(P)], I),
        "qk_simulate": ([P, P, C.POINTER(_Config), U64, C.POINTER(_RunStats)], I),
        "qk_simulate_local": ([C.POINTER(P), I, P, C.POINTER(_Config), U64, C.POINTER(_XrsStats)], I),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc:
        raise _ERRORS.get(rc, SimulationError)(lib().qk_last_error().decode())


def _text(fn, *args) -> str:
    out = C.c_void_p()
    _check(fn(*args, C.byref(out)))
    s = C.cast(out, C.c_char_p).value.decode()
    lib().qk_free(out)
    return s


def device_count() -> int:
    n = C.c_int(0)
    _check(lib().qk_device_count(C.byref(n)))
    return n.value


# ---------------------------------------------------------------- config

class Config:
    """The reference's [system] INI config (proj/src/circuit.cpp:489-545)."""

    FIELDS = ("total_qubits", "rank_qubits", "buffer_qubits", "chunk_qubits", "fusion_qubits",
              "cache_line_qubits", "ims", "xrs", "fusion", "diagonal_fusion")

    def __init__(self, c: _Config):
        self._c = c

    @classmethod
    def parse(cls, text: str) -> "Config":
        c = _Config()
        _check(lib().qk_config_parse(text.encode(), C.byref(c)))
        return cls(c)

    @classmethod
    def make(cls, n, r=0, chunk=-1, fusion_qubits=-1, buffer=-1, cache_line=-1, ims=1, xrs=1,
             fusion=1, diag=1) -> "Config":
        c = _Config(n, r, buffer, chunk, fusion_qubits, cache_line, ims, xrs, fusion, diag)
        _check(lib().qk_config_finalize(C.byref(c)))
        return cls(c)

    @classmethod
    def tune(cls, circuit_text: str, n: int, r: int = 0, hbm_bytes: float = 0.0):
        """GPU-aware configuration: (Config, report) -- the candidate whose
        reference-optimizer Program this engine runs cheapest (qk_config_tune)."""
        c = _Config()
        rep = C.c_void_p()
        _check(lib().qk_config_tune(circuit_text.encode(), n, r, hbm_bytes, C.byref(c), C.byref(rep)))
        text = C.cast(rep, C.c_char_p).value.decode()
        lib().qk_free(rep)
        return cls(c), text

    def __getattr__(self, k):
        if k in Config.FIELDS:
            return getattr(self._c, k)
        raise AttributeError(k)

    def text(self) -> str:
        return _text(lib().qk_config_serialize, C.byref(self._c))


# ---------------------------------------------------------------- programs

class Program:
    """A parsed (SQS/CSQS program text) or AIO-optimized Program."""

    def __init__(self, handle, cfg: Config):
        self._h = C.c_void_p(handle)
        self.cfg = cfg

    @classmethod
    def parse(cls, text: str, cfg: Config, lenient: bool = False) -> "Program":
        h = C.c_void_p()
        _check(lib().qk_program_parse(text.encode(), C.byref(cfg._c), int(lenient), C.byref(h)))
        return cls(h.value, cfg)

    @classmethod
    def optimize(cls, circuit_text: str, cfg: Config) -> "Program":
        """aioOptimize (proj/src/optimizer.cpp:478-485), this framework's host C++."""
        h = C.c_void_p()
        _check(lib().qk_program_optimize(circuit_text.encode(), C.byref(cfg._c), C.byref(h)))
        return cls(h.value, cfg)

    def text(self) -> str:
        return _text(lib().qk_program_serialize, self._h)

    def debug_compile(self, n_local: int | None = None) -> dict:
        """Device item list the engine runs (host only; test hook)."""
        import json
        n_local = self.cfg.total_qubits - self.cfg.rank_qubits if n_local is None else n_local
        return json.loads(_text(lib().qk_debug_compile_program, self._h, n_local))

    def debug_jit_sources(self, n_local: int | None = None) -> list:
        """[(name, CUDA source)] of every specialized pass kernel (host only; test hook)."""
        n_local = self.cfg.total_qubits - self.cfg.rank_qubits if n_local is None else n_local
        out = []
        for chunk in _text(lib().qk_debug_jit_program, self._h, n_local).split("//@@PASS ")[1:]:
            name, src = chunk.split("\n", 1)
            out.append((name.strip(), src))
        return out

    def counts(self):
        v = [C.c_int64() for _ in range(4)]
        _check(lib().qk_program_counts(self._h, *[C.byref(x) for x in v]))
        return dict(zip(("blocks", "sqs", "csqs", "gates"), (x.value for x in v)))

    def final_layout(self):
        n = self.cfg.total_qubits
        arr = (C.c_int * n)()
        _check(lib().qk_program_final_layout(self._h, arr))
        return list(arr)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None:
            _lib.qk_program_destroy(self._h)
            self._h = C.c_void_p()


def generate(kind: str, n: int, a: int = 0, seed: int = 0) -> str:
    """Circuit text from the generators (tools.cpp:169-272, + grover)."""
    return _text(lib().qk_circuit_generate, kind.encode(), n, a, seed)


def circuit_roundtrip(text: str, n: int = -1) -> str:
    return _text(lib().qk_circuit_roundtrip, text.encode(), n)


# ---------------------------------------------------------------- device state

class State:
    """One rank slice of 2^(n-r) complex128 amplitudes resident in HBM."""

    def __init__(self, n: int, r: int = 0, rank: int = 0, buffer: int = -1, device: int = 0):
        h = C.c_void_p()
        _check(lib().qk_create(n, r, rank, buffer, device, C.byref(h)))
        self._h = h
        self.n, self.r, self.rank = n, r, rank
        self.count = 1 << (n - r)

    def close(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None:
            _lib.qk_destroy(self._h)
            self._h = C.c_void_p()

    __del__ = close

    def set_basis(self, index: int) -> None:
        _check(lib().qk_set_basis(self._h, index))

    def upload(self, amps: np.ndarray, offset: int = 0) -> None:
        a = np.ascontiguousarray(amps, dtype=np.complex128)
        _check(lib().qk_upload(self._h, offset, a.size, a.ctypes.data))

    def download(self, offset: int = 0, count: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
        count = self.count - offset if count is None else count
        if out is None:
            out = np.empty(count, dtype=np.complex128)
        _check(lib().qk_download(self._h, offset, count, out.ctypes.data))
        return out

    def stream_chunks(self, fn, offset: int = 0, count: int | None = None, chunk: int = 1 << 22) -> None:
        """Stream [offset, offset + count) to fn(ndarray complex128 chunk) through
        two pinned buffers (qk_download_stream): for states larger than host RAM."""
        count = self.count - offset if count is None else count
        err = []

        def sink(ptr, n, _user):
            try:
                fn(np.ctypeslib.as_array(ptr, shape=(2 * n,)).view(np.complex128))
                return 0
            except Exception as e:  # noqa: BLE001
                err.append(e)
                return 1
        cb = _SINK(sink)
        rc = lib().qk_download_stream(self._h, offset, count, chunk, cb, None)
        if err:
            raise err[0]
        _check(rc)

    def save(self, path: str, chunk: int = 1 << 22) -> None:
        """Write the slice (physical order, interleaved complex128) to a file, streamed."""
        with open(path, "wb") as f:
            self.stream_chunks(lambda a: f.write(a.tobytes()), chunk=chunk)

    def norm(self) -> float:
        v = C.c_double()
        _check(lib().qk_norm(self._h, C.byref(v)))
        return v.value

    def marginal(self, bits) -> np.ndarray:
        """Probabilities over the given slice bits (physical positions): 2^k values."""
        arr = (C.c_int * max(1, len(bits)))(*bits)
        out = np.empty(1 << len(bits), dtype=np.float64)
        _check(lib().qk_marginal(self._h, arr, len(bits), out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def synchronize(self) -> None:
        _check(lib().qk_synchronize(self._h))

    def stream(self) -> int:
        s = C.c_void_p()
        _check(lib().qk_stream(self._h, C.byref(s)))
        return s.value or 0

    def set_profiling(self, on: bool) -> None:
        _check(lib().qk_set_profiling(self._h, int(on)))

    def comm_init(self, unique_id: bytes, nranks: int, rank: int) -> None:
        _check(lib().qk_comm_init(self._h, unique_id, nranks, rank))

    def ipc_init(self, job: str, nranks: int, rank: int) -> None:
        """Join the node-local peer-memory rank group `job` (collective): CSQS
        items then run as in-place swaps over the mapped peer slices."""
        _check(lib().qk_ipc_init(self._h, job.encode(), nranks, rank))

    def simulate(self, prog: Program, initial: int = 0) -> dict:
        rs = _RunStats()
        _check(lib().qk_simulate(self._h, prog._h, C.byref(prog.cfg._c), initial, C.byref(rs)))
        return {k: getattr(rs, k) for k, _ in _RunStats._fields_}

    def xrs_swap(self, pairs):
        """Multi-process XRS over this rank's group (peer memory if ipc_init, else NCCL)."""
        outs, ins, s = _pairs(pairs)
        st = _XrsStats()
        _check(lib().qk_xrs_swap(self._h, outs, ins, s, C.byref(st)))
        return (st.bytes_sent, st.bytes_received, st.peak_buffer_bytes, st.rounds)


def xrs_plan(n: int, r: int, buffer: int, rank: int, pairs):
    """This rank's XRS message schedule (host-only; what the NCCL path executes)."""
    outs, ins, s = _pairs(pairs)
    cap = 1 << 16
    msgs = (_XrsMsg * cap)()
    nm = C.c_int()
    _check(lib().qk_xrs_plan(n, r, buffer, rank, outs, ins, s, msgs, cap, C.byref(nm)))
    return [{k: getattr(m, k) for k, _ in _XrsMsg._fields_} for m in msgs[:nm.value]]


def xrs_slab_index(n: int, r: int, outs, slab: int, offset: int) -> int:
    """Slice index of element `offset` of slab `slab` (distributed.cpp:65-71)."""
    arr = (C.c_int * max(1, len(outs)))(*outs)
    out = C.c_uint64()
    _check(lib().qk_xrs_slab_index(n, r, arr, len(outs), slab, offset, C.byref(out)))
    return out.value


def debug_host_barrier(job: str, nranks: int, rank: int, rounds: int, timeout_s: float = 60.0) -> None:
    """Pass qk_ipc_init's shared-memory barrier `rounds` times (host-only test hook)."""
    _check(lib().qk_debug_host_barrier(job.encode(), nranks, rank, rounds, timeout_s))


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().qk_comm_unique_id(buf))
    return buf.raw


# ---------------------------------------------------------------- gates

class Gate:
    """One gate in the reference's matrix order (controls first; first = MSB)."""

    def __init__(self, kind: str, qubits, params=(), payload=None, gid: int = -1):
        self.kind, self.qubits, self.params, self.gid = kind, list(qubits), list(params), gid
        self.payload = None if payload is None else np.ascontiguousarray(payload, dtype=np.float64)

    @classmethod
    def parse(cls, line: str) -> "Gate":
        """Gate line of the program format (proj/src/circuit.cpp:176-274)."""
        toks = line.split("#")[0].split("//")[0].split()
        k = toks[0]
        if len(k) >= 2 and k[0] in "DU" and k[1:].isdigit():
            n = int(k[1:])
            qs = [int(t) for t in toks[1:1 + n]]
            ent = (1 << n) if k[0] == "D" else (1 << (2 * n))
            vals = [float(t) for t in toks[1 + n:1 + n + 2 * ent]]
            return cls("D" if k[0] == "D" else "UK", qs, payload=vals)
        arity = 2 if k in ("CX", "CP", "SWAP", "RZZ") else 1
        qs = [int(t) for t in toks[1:1 + arity]]
        gid = int(toks[1 + arity])
        return cls(k, qs, [float(t) for t in toks[2 + arity:]], gid=gid)

    def _fill(self, g: _Gate):
        g.kind = KINDS[self.kind]
        g.nqubits = len(self.qubits)
        for j, q in enumerate(self.qubits):
            g.qubits[j] = q
        for j, p in enumerate(self.params[:3]):
            g.params[j] = p
        if self.payload is not None:
            g.payload = self.payload.ctypes.data_as(C.POINTER(C.c_double))
        g.id = self.gid


def _gate_array(gates):
    gs = [g if isinstance(g, Gate) else Gate.parse(g) for g in gates]
    arr = (_Gate * max(1, len(gs)))()
    for i, g in enumerate(gs):
        g._fill(arr[i])
    return arr, gs


def _pairs(pairs):
    s = len(pairs)
    outs = (C.c_int * max(1, s))(*[p[0] for p in pairs])
    ins = (C.c_int * max(1, s))(*[p[1] for p in pairs])
    return outs, ins, s


# ---------------------------------------------------------------- reference-shaped API

def apply_block(state: State, gates, chunk_qubits: int) -> None:
    """applyBlock (engine.cpp:262-281) on a device slice."""
    arr, keep = _gate_array(gates)
    _check(lib().qk_apply_block(state._h, arr, len(keep), chunk_qubits))


def debug_compile_block(gates, n_local: int) -> dict:
    """The scheduler's pass programs for a block (host only; test hook)."""
    import json
    arr, keep = _gate_array(gates)
    return json.loads(_text(lib().qk_debug_compile_block, arr, len(keep), n_local))


def set_jit_min_qubits(v: int) -> None:
    """Slices with >= v local qubits use straight-line specialized pass kernels."""
    _check(lib().qk_set_jit_min_qubits(v))


def debug_jit_compile(gates, n_local: int) -> str:
    """Generate and NVRTC-compile a block's specialized kernels (host only)."""
    arr, keep = _gate_array(gates)
    return _text(lib().qk_debug_jit_compile, arr, len(keep), n_local)


def apply_gate(state: State, gate) -> None:
    arr, keep = _gate_array([gate])
    _check(lib().qk_apply_gate(state._h, arr))


def ims_swap(state: State, pairs, cache_line_qubits: int = 2) -> None:
    """imsSwap (engine.cpp:86-101) on a device slice."""
    outs, ins, s = _pairs(pairs)
    _check(lib().qk_ims_swap(state._h, outs, ins, s, cache_line_qubits))


def set_ims_mode(mode: int) -> None:
    """IMS kernel choice: 0 per-element, 1 tiled when possible (default), 2 tiled
    only for pairs moving memory bit 0/1."""
    _check(lib().qk_set_ims_mode(mode))


def set_dense_mode(mode: int) -> None:
    """Fused U5 kernel: 0 DFMA, 1 DMMA (FP64 tensor cores), -1 autotune (default)."""
    _check(lib().qk_set_dense_mode(mode))


def xrs_swap(slices, pairs):
    """xrsSwap (distributed.cpp:124-138) over slices owned by this process."""
    outs, ins, s = _pairs(pairs)
    arr = (C.c_void_p * len(slices))(*[x._h.value for x in slices])
    stats = (_XrsStats * len(slices))()
    _check(lib().qk_xrs_swap_local(arr, len(slices), outs, ins, s, stats))
    return [(x.bytes_sent, x.bytes_received, x.peak_buffer_bytes, x.rounds) for x in stats]


def xrs_swap_loopback(slices, pairs):
    """The NCCL path's per-rank XRS schedule (pack / single receive buffer /
    copy-back) for slices in this process, transfers as device copies."""
    outs, ins, s = _pairs(pairs)
    arr = (C.c_void_p * len(slices))(*[x._h.value for x in slices])
    stats = (_XrsStats * len(slices))()
    _check(lib().qk_xrs_swap_loopback(arr, len(slices), outs, ins, s, stats))
    return [(x.bytes_sent, x.bytes_received, x.peak_buffer_bytes, x.rounds) for x in stats]


def simulate_program(prog: Program, initial: int = 0, device: int = 0):
    """simulateProgram (engine.cpp:283-297): returns (state ndarray, physToLog)."""
    st = State(prog.cfg.total_qubits, 0, 0, prog.cfg.buffer_qubits, device)
    try:
        st.simulate(prog, initial)
        return st.download(), prog.final_layout()
    finally:
        st.close()


def spawn_ranks(prog: Program, initial: int = 0, device: int = 0):
    """spawnRanks (distributed.cpp:140-206) with all 2^R slices in this process.

    Returns (gathered state, physToLog, per-rank stats)."""
    cfg = prog.cfg
    ranks = 1 << cfg.rank_qubits
    sl = [State(cfg.total_qubits, cfg.rank_qubits, k, cfg.buffer_qubits, device) for k in range(ranks)]
    try:
        arr = (C.c_void_p * ranks)(*[x._h.value for x in sl])
        stats = (_XrsStats * ranks)()
        _check(lib().qk_simulate_local(arr, ranks, prog._h, C.byref(cfg._c), initial, stats))
        state = np.concatenate([x.download() for x in sl])
        return state, prog.final_layout(), [(s.bytes_sent, s.bytes_received, s.peak_buffer_bytes,
                                             s.rounds) for s in stats]
    finally:
        for x in sl:
            x.close()
