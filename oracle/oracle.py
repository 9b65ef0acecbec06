"""TEST INFRASTRUCTURE ONLY — Python handle on the CPU oracles.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module, and only as the checker or
the timed CPU baseline — never as the thing measured on the GPU path.

Two oracles live here:

* ``Ref``   — ``_ref/libquokka_ref.so``: the UNMODIFIED reference (Quokka,
  ``/root/reference/proj/src``) compiled from its own sources with the
  namespace renamed, behind ``ref_shim.cpp``'s C-ABI.
* ``Port``  — ``_ref/libqk_oracle.so``: ``quokka_oracle.c``, the plain-C
  restatement of the reference's hot-path arithmetic (bit-exact to ``Ref``;
  pinned by tests/test_oracle.py).

Gate-line parsing for the restatement follows proj/src/circuit.cpp:176-274.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

KINDS = {"H": 0, "U": 1, "X": 2, "CX": 3, "CP": 4, "SWAP": 5, "RX": 6, "RY": 7,
         "RZ": 8, "RZZ": 9}
ARITY = {"H": 1, "U": 1, "X": 1, "CX": 2, "CP": 2, "SWAP": 2, "RX": 1, "RY": 1,
         "RZ": 1, "RZZ": 2}
NPARAM = {"H": 0, "U": 3, "X": 0, "CX": 0, "CP": 1, "SWAP": 0, "RX": 1, "RY": 1,
          "RZ": 1, "RZZ": 1}


def build() -> None:
    """Compile the oracles (make -C oracle). The reference .so only builds
    where /root/reference exists; elsewhere the prebuilt file is used."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class _Gate(C.Structure):
    _fields_ = [("kind", C.c_int), ("nq", C.c_int), ("q", C.c_int * 16),
                ("p", C.c_double * 3), ("payload", C.POINTER(C.c_double))]


def parse_gate_line(line: str):
    """(kind, qubits-in-matrix-order, params, payload ndarray|None)."""
    toks = line.split("#")[0].split("//")[0].split()
    k = toks[0]
    if len(k) >= 2 and k[0] in "DU" and k[1:].isdigit():
        n = int(k[1:])
        qs = [int(t) for t in toks[1:1 + n]]
        ent = (1 << n) if k[0] == "D" else (1 << (2 * n))
        vals = np.array([float(t) for t in toks[1 + n:1 + n + 2 * ent]], dtype=np.float64)
        return ("D" if k[0] == "D" else "UK"), qs, [], vals
    a = ARITY[k]
    qs = [int(t) for t in toks[1:1 + a]]
    params = [float(t) for t in toks[2 + a:]]
    params += [0.0] * (NPARAM[k] - len(params))
    return k, qs, params, None


class Port:
    """ctypes facade over quokka_oracle.c."""

    def __init__(self):
        self.lib = C.CDLL(os.path.join(REF_DIR, "libqk_oracle.so"))
        L = self.lib
        L.qo_apply_block.argtypes = [C.c_void_p, C.c_int, C.POINTER(_Gate), C.c_int, C.c_int]
        L.qo_apply_gate.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(_Gate)]
        L.qo_ims_swap.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int]
        L.qo_xrs_swap.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int),
                                  C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_uint64)]
        L.qo_bitswap.argtypes = [C.c_uint64, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int]
        L.qo_bitswap.restype = C.c_uint64
        L.qo_norm.argtypes = [C.c_void_p, C.c_uint64]
        L.qo_norm.restype = C.c_double
        L.qo_init.argtypes = [C.c_void_p, C.c_int, C.c_uint64]

    @staticmethod
    def gates_of(lines):
        keep = []
        arr = (_Gate * max(1, len(lines)))()
        for i, ln in enumerate(lines):
            kind, qs, params, payload = parse_gate_line(ln)
            g = arr[i]
            g.kind = {"D": 10, "UK": 11}.get(kind, KINDS.get(kind, -1))
            g.nq = len(qs)
            for j, q in enumerate(qs):
                g.q[j] = q
            for j, p in enumerate(params[:3]):
                g.p[j] = p
            if payload is not None:
                payload = np.ascontiguousarray(payload)
                keep.append(payload)
                g.payload = payload.ctypes.data_as(C.POINTER(C.c_double))
        return arr, keep

    def apply_block(self, state: np.ndarray, n: int, lines, chunk: int) -> None:
        arr, keep = self.gates_of(lines)
        rc = self.lib.qo_apply_block(state.ctypes.data, n, arr, len(lines), chunk)
        if rc:
            raise ValueError("block gate reaches outside the chunk")

    def ims_swap(self, state: np.ndarray, n: int, pairs) -> None:
        outs = (C.c_int * len(pairs))(*[p[0] for p in pairs])
        ins = (C.c_int * len(pairs))(*[p[1] for p in pairs])
        self.lib.qo_ims_swap(state.ctypes.data, n, outs, ins, len(pairs))

    def xrs_swap(self, state: np.ndarray, n: int, r: int, b: int, pairs):
        s = len(pairs)
        outs = (C.c_int * max(1, s))(*[p[0] for p in pairs])
        ins = (C.c_int * max(1, s))(*[p[1] for p in pairs])
        stats = np.zeros(4 << r, dtype=np.uint64)
        rc = self.lib.qo_xrs_swap(state.ctypes.data, n, r, b, outs, ins, s,
                                  stats.ctypes.data_as(C.POINTER(C.c_uint64)))
        if rc:
            raise ValueError("invalid cross-rank swap")
        return stats.reshape(-1, 4)

    def run_program(self, text: str, n: int, chunk: int, initial: int = 0) -> np.ndarray:
        """simulateProgram restated (engine.cpp:283-297): single rank, SQS items
        via imsSwap, blocks via applyBlock.  Record parsing per circuit.cpp:394-460."""
        state = self.init(n, initial)
        lines = [ln.split("#")[0].split("//")[0].strip() for ln in text.splitlines()]
        lines = [ln for ln in lines if ln]
        i = 0
        while i < len(lines):
            head = lines[i].split()
            if head[0] in ("SQS", "CSQS"):
                body, i = [lines[i]], i + 1
            else:
                k = int(head[0])
                body, i = lines[i + 1:i + 1 + k], i + 1 + k
            if body[0].startswith("CSQS"):
                raise ValueError("cross-rank swap in a single-rank run")
            if body[0].startswith("SQS"):
                t = body[0].split()
                s = int(t[1])
                self.ims_swap(state, n, list(zip(map(int, t[2:2 + s]), map(int, t[2 + s:]))))
            else:
                self.apply_block(state, n, body, chunk)
        return state

    def norm(self, state: np.ndarray) -> float:
        return self.lib.qo_norm(state.ctypes.data, state.size // 2)

    def init(self, n: int, initial: int = 0) -> np.ndarray:
        a = np.empty(2 << n, dtype=np.float64)
        self.lib.qo_init(a.ctypes.data, n, initial)
        return a


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Ref:
    """ctypes facade over the reference build (ref_shim.cpp)."""

    def __init__(self):
        path = os.path.join(REF_DIR, "libquokka_ref.so")
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_free.argtypes = [C.c_void_p]
        cp = C.POINTER(C.c_char_p)
        L.ref_gen.argtypes = [C.c_char_p, C.c_int, C.c_long, C.c_ulonglong, C.POINTER(C.c_void_p)]
        L.ref_optimize.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]
        L.ref_program_roundtrip.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_circuit_roundtrip.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_config_roundtrip.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.ref_simulate.argtypes = [C.c_char_p, C.c_char_p, C.c_ulonglong, C.c_int, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]
        L.ref_run_items.argtypes = [C.c_char_p, C.c_char_p, C.c_void_p, C.c_int, C.c_int,
                                    C.c_int, C.POINTER(C.c_double)]
        L.ref_apply_block.argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.c_int, C.c_int]
        L.ref_apply_gate.argtypes = [C.c_void_p, C.c_int, C.c_char_p]
        L.ref_ims_swap.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                   C.c_int, C.c_int, C.c_int]
        L.ref_bitswap.argtypes = [C.c_ulonglong, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int]
        L.ref_bitswap.restype = C.c_ulonglong
        L.ref_bitshift.argtypes = [C.c_ulonglong, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int,
                                   C.c_int]
        L.ref_bitshift.restype = C.c_ulonglong
        L.ref_xrs_swap.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int),
                                   C.POINTER(C.c_int), C.c_int, C.c_void_p]
        L.ref_oracle_simulate.argtypes = [C.c_char_p, C.c_int, C.c_ulonglong, C.c_void_p]
        L.ref_layout_apply.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int)]
        L.ref_validate_order.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p]
        del cp

    def _check(self, rc):
        if rc:
            raise RefError(rc, self.lib.ref_last_error().decode())

    def _text(self, fn, *args) -> str:
        out = C.c_void_p()
        self._check(fn(*args, C.byref(out)))
        s = C.cast(out, C.c_char_p).value.decode()
        self.lib.ref_free(out)
        return s

    def gen(self, kind: str, n: int, a: int = 0, seed: int = 0) -> str:
        return self._text(self.lib.ref_gen, kind.encode(), n, a, seed)

    def optimize(self, circuit: str, cfg: str) -> str:
        return self._text(self.lib.ref_optimize, circuit.encode(), cfg.encode())

    def program_roundtrip(self, prog: str, cfg: str, lenient=False) -> str:
        return self._text(self.lib.ref_program_roundtrip, prog.encode(), cfg.encode(), int(lenient))

    def circuit_roundtrip(self, text: str, n: int = -1) -> str:
        return self._text(self.lib.ref_circuit_roundtrip, text.encode(), n)

    def config_roundtrip(self, text: str) -> str:
        return self._text(self.lib.ref_config_roundtrip, text.encode())

    def simulate(self, prog: str, cfg: str, n: int, r: int = 0, initial: int = 0, threads: int = 0):
        """Returns (state[2^n complex], physToLog, stats|None, seconds)."""
        state = np.empty(2 << n, dtype=np.float64)
        p2l = (C.c_int * n)()
        stats = np.zeros(4 << r, dtype=np.uint64)
        sec = C.c_double()
        self._check(self.lib.ref_simulate(prog.encode(), cfg.encode(), initial, threads,
                                          state.ctypes.data, p2l, stats.ctypes.data, C.byref(sec)))
        return state, list(p2l), (stats.reshape(-1, 4) if r else None), sec.value

    def run_items(self, prog: str, cfg: str, state: np.ndarray, first: int, last: int,
                  threads: int = 0) -> float:
        sec = C.c_double()
        self._check(self.lib.ref_run_items(prog.encode(), cfg.encode(), state.ctypes.data,
                                           first, last, threads, C.byref(sec)))
        return sec.value

    def apply_block(self, state: np.ndarray, n: int, lines, chunk: int, threads: int = 1):
        self._check(self.lib.ref_apply_block(state.ctypes.data, n, "\n".join(lines).encode(),
                                             chunk, threads))

    def apply_gate(self, state: np.ndarray, n: int, line: str):
        self._check(self.lib.ref_apply_gate(state.ctypes.data, n, line.encode()))

    def ims_swap(self, state: np.ndarray, n: int, pairs, cl: int = 2, threads: int = 1):
        s = len(pairs)
        outs = (C.c_int * s)(*[p[0] for p in pairs])
        ins = (C.c_int * s)(*[p[1] for p in pairs])
        self._check(self.lib.ref_ims_swap(state.ctypes.data, n, outs, ins, s, cl, threads))

    def bitswap(self, x: int, pairs) -> int:
        s = len(pairs)
        outs = (C.c_int * max(1, s))(*[p[0] for p in pairs])
        ins = (C.c_int * max(1, s))(*[p[1] for p in pairs])
        return self.lib.ref_bitswap(x, outs, ins, s)

    def xrs_swap(self, state: np.ndarray, n: int, r: int, b: int, pairs):
        s = len(pairs)
        outs = (C.c_int * max(1, s))(*[p[0] for p in pairs])
        ins = (C.c_int * max(1, s))(*[p[1] for p in pairs])
        stats = np.zeros(4 << r, dtype=np.uint64)
        self._check(self.lib.ref_xrs_swap(state.ctypes.data, n, r, b, outs, ins, s,
                                          stats.ctypes.data))
        return stats.reshape(-1, 4)

    def oracle_simulate(self, circuit: str, n: int, initial: int = 0) -> np.ndarray:
        state = np.empty(2 << n, dtype=np.float64)
        self._check(self.lib.ref_oracle_simulate(circuit.encode(), n, initial, state.ctypes.data))
        return state

    def layout_apply(self, state: np.ndarray, n: int, phys_to_log) -> np.ndarray:
        out = state.copy()
        p2l = (C.c_int * n)(*phys_to_log)
        self._check(self.lib.ref_layout_apply(out.ctypes.data, n, p2l))
        return out

    def validate_order(self, circuit: str, prog: str, cfg: str) -> bool:
        rc = self.lib.ref_validate_order(circuit.encode(), prog.encode(), cfg.encode())
        if rc < 0:
            raise RefError(-rc, self.lib.ref_last_error().decode())
        return rc == 1


def config_text(n, r=0, c=None, f=None, b=None, cl=None, ims=1, xrs=1, fusion=1, diag=1) -> str:
    """INI text in the reference's [system] format (circuit.cpp:489-545)."""
    lines = ["[system]", f"total_qbit={n}", f"rank_qbit={r}"]
    if b is not None:
        lines.append(f"buffer_qbit={b}")
    if c is not None:
        lines.append(f"chunk_qbit={c}")
    if f is not None:
        lines.append(f"fusion_qbit={f}")
    if cl is not None:
        lines.append(f"cache_line_qbit={cl}")
    lines += [f"ims={ims}", f"xrs={xrs}", f"fusion={fusion}", f"diagonal_fusion={diag}"]
    return "\n".join(lines) + "\n"


def random_state(n: int, seed: int) -> np.ndarray:
    """Same RNG stream as the reference tests' randomState
    (proj/tests/test_engine.cpp:20-31; Rng at proj/include/quokka/common.hpp:32-66)."""
    M = (1 << 64) - 1

    def splitmix(x):
        x = (x + 0x9E3779B97F4A7C15) & M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
        return x ^ (x >> 31)

    size = 1 << n
    st = splitmix(seed)
    raw = np.empty(2 * size, dtype=np.uint64)
    for i in range(2 * size):
        x = st
        x ^= x >> 12
        x ^= (x << 25) & M
        x ^= x >> 27
        st = x
        raw[i] = (x * 0x2545F4914F6CDD1D) & M
    d = (raw >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 - 0.5
    norm = 0.0
    for i in range(size):  # same sequential summation order as the reference
        norm += d[2 * i] * d[2 * i] + d[2 * i + 1] * d[2 * i + 1]
    norm = np.sqrt(norm)
    return d / norm
