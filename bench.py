#!/usr/bin/env python3
"""Benchmark: QFT state-vector simulation, weak-scaled 2^33 amplitudes per GPU
(33 qubits @ 1 GPU ... 36 qubits @ 8 GPUs), BASELINE.json's headline metric
"circuit sim time (s)".

One step = one full simulation of the program (initState + every block / IMS /
XRS item) on resident HBM state — exactly what the reference times
(proj/tools/main.cpp:126-145: wall from initState to the last item; parse and
optimize excluded).  Lower is better.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one process per GPU)

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "circuit sim time (s) and roofline fraction, 33q@1 GPU to 36q@8 GPU vs CPU ref"
PER_GPU_QUBITS = 33


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--circuit", default="qft", help="qft | bvones | qaoa | random | grover")
    ap.add_argument("--per-gpu-qubits", type=int, default=PER_GPU_QUBITS)
    ap.add_argument("--chunk", type=int, default=13)
    ap.add_argument("--cpu-sample-qubits", type=int, default=28,
                    help="measured reference run for cpu_baseline (same-size GPU/CPU pair)")
    ap.add_argument("--ref-sample-qubits", type=int, default=26,
                    help="--impl reference: per-step reference sample size")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def circuit_args(kind, n):
    return {"qft": (0, 0), "bvones": (0, 0), "qaoa": (1, 1), "random": (400, 7), "grover": (1, 5)}[kind]


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.proc = None
        self.gpu = gpu_index
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
            return self
        # nvidia-smi takes a moment to start: time only once it is sampling
        t0 = time.time()
        while time.time() - t0 < 5.0 and self.proc.poll() is None:
            self.fh.flush()
            if os.path.getsize(self.path) > 0:
                break
            time.sleep(0.02)
        self.start = os.path.getsize(self.path)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        with open(self.path) as f:
            f.seek(getattr(self, "start", 0))
            lines = f.read().splitlines()
        for line in lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8 and parts[0].replace(".", "").isdigit():
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(float(r[0]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())}


# ------------------------------------------------------------------ peaks

def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


def ncu_traffic():
    path = os.path.join(ROOT, "profiles", "block_pass_traffic.json")
    if os.path.exists(path):
        return json.load(open(path))
    return None


# ------------------------------------------------------------------ CPU baseline

def ref_circuit(ref, kind, n):
    """Circuit text for the reference path.  The reference's own generators
    (tools.cpp:169-272) for its kinds; Grover (which the reference lacks, its
    tools.hpp:38-48) is written by a separate process so that the process
    timing the reference never loads this repo's library."""
    a, seed = circuit_args(kind, n)
    if kind != "grover":
        return ref.gen(kind, n, a, seed)
    code = ("import sys; sys.path.insert(0, %r); import paper_2409_14697_b200 as qk; "
            "sys.stdout.write(qk.generate('grover', %d, %d, %d))" % (ROOT, n, a, seed))
    return subprocess.run([sys.executable, "-c", code], check=True, capture_output=True, text=True).stdout


def program_items(text):
    """Items (blocks + SQS + CSQS) of a program text (circuit.cpp:394-460)."""
    lines = [ln for ln in text.splitlines() if ln.strip()]
    items = i = 0
    while i < len(lines):
        k = int(lines[i].split()[0])
        items += 1
        i += 1 + k
    return items


def cpu_reference_run(kind, n, chunk, threads, initial=0):
    """The reference's simulateProgram (oracle/_ref: /root/reference/proj/src
    compiled unmodified) on an n-qubit program with `threads` host threads.
    Timed region = initState .. last item (proj/tools/main.cpp:126-145); the
    shim's copy-out of the state is outside it.  Returns (seconds, items)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Ref, config_text
    ref = Ref()
    cfg = config_text(n, 0, min(chunk, n), fusion=0, diag=0)
    prog = ref.optimize(ref_circuit(ref, kind, n), cfg)
    _, _, _, sec = ref.simulate(prog, cfg, n, 0, initial, threads)
    return sec, program_items(prog), prog


def extrapolate(kind, n_sample, sec, items_sample, n_target, chunk, R=0):
    """Scale a measured reference run to the target size by amplitude-passes:
    every reference item (applyBlock / imsSwap, engine.cpp:262-297) sweeps the
    whole state once, so its time is linear in 2^n x items."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Ref, config_text
    ref = Ref()
    cfg = config_text(n_target, 0, chunk, fusion=0, diag=0)
    items_t = program_items(ref.optimize(ref_circuit(ref, kind, n_target), cfg))
    scale = (2.0 ** n_target * items_t) / (2.0 ** n_sample * items_sample)
    return sec * scale, scale, items_t


# ------------------------------------------------------------------ main

def spawn_ranks_self(args):
    """`python bench.py --gpus N` without torchrun: launch N ranks (one process
    per GPU) through torch.distributed.run on 127.0.0.1 and pass on the exit code."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} needs {args.gpus} visible GPUs, "
                                                     f"found {have} (one process per GPU, 2^{args.per_gpu_qubits} "
                                                     "amplitudes each)"}), flush=True)
        return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if args.impl == "reference":
            world = 1  # the reference arm runs on rank 0's host cores only
        else:
            sys.exit(spawn_ranks_self(args))
    if world > 1:
        args.gpus = world
    R = int(round(math.log2(max(1, args.gpus))))
    n = args.per_gpu_qubits + R
    kind = args.circuit

    if args.impl == "reference":
        return run_reference(args, rank, n, R, kind)

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2409_14697_b200 as qk

    # QK_BENCH_SHARE_GPU=1 (test hook): every rank on cuda:0 with a gloo
    # process group -- the multi-rank path (peer-memory XRS) on a 1-GPU box.
    share = os.environ.get("QK_BENCH_SHARE_GPU") == "1"
    device = 0 if share else local_rank
    torch.cuda.set_device(device)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    tdev = "cpu" if share else "cuda"

    a, seed = circuit_args(kind, n)
    circ = qk.generate(kind, n, a, seed)
    cfg = qk.Config.make(n, R, chunk=args.chunk, fusion=0, diag=0)
    t0 = time.perf_counter()
    prog = qk.Program.optimize(circ, cfg)
    opt_s = time.perf_counter() - t0
    counts = prog.counts()
    prog_text = prog.text()

    st = qk.State(n, R, rank, cfg.buffer_qubits, device)
    # Cross-rank transport: the peer-memory rank group (qk_ipc_init: one
    # in-place swap kernel per CSQS over NVLink P2P, no buffer, no copy-back)
    # is the default -- it is the path exercised on hardware (multi-process
    # tests on the B200); QK_XRS=nccl selects grouped ncclSend/ncclRecv.
    transport = os.environ.get("QK_XRS", "ipc")
    if world > 1 and transport == "ipc":
        # peer-memory rank group: in-place swap kernels over NVLink, no buffer
        job = [f"bench{os.getpid()}_{time.time_ns()}" if rank == 0 else None]
        dist.broadcast_object_list(job, 0)
        st.ipc_init(job[0], world, rank)
    elif world > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device=tdev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(qk.comm_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        st.comm_init(bytes(uid.cpu().numpy().tobytes()), world, rank)

    ext = torch.cuda.ExternalStream(st.stream())

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # Cold first call of a new program: NVRTC specialization of every pass,
    # table upload and the first autotune run (wall clock, synchronous).
    barrier()
    t1 = time.perf_counter()
    tuning = st.simulate(prog, 0)["tuning_runs"]
    cold_s = time.perf_counter() - t1
    # Schedule autotune (register widths per pass, tile size per gate stream)
    # settles over the first few runs of a program; finish it before the
    # warm-up so the timed steps run the tuned schedule.
    # Every rank must call simulate equally often (each CSQS is a collective):
    # a rank keeps going while ANY rank is still tuning (the rank holding
    # |initial> times passes the others skip).
    def any_tuning(x):
        if world == 1:
            return bool(x)
        f = torch.tensor([float(x)], dtype=torch.float64, device=tdev)
        dist.all_reduce(f, op=dist.ReduceOp.MAX)
        return bool(f.item())

    tune_runs = 1
    tuning = any_tuning(tuning)
    while tune_runs < 24 and tuning:
        tuning = any_tuning(st.simulate(prog, 0)["tuning_runs"])
        tune_runs += 1
    for _ in range(args.warmup):
        st.simulate(prog, 0)
    barrier()

    st.set_profiling(True)
    stats = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device) as clk:
        barrier()
        ev0.record(ext)
        for _ in range(args.steps):
            stats.append(st.simulate(prog, 0))
        ev1.record(ext)
        barrier()
    st.set_profiling(False)
    dev_ms = ev0.elapsed_time(ev1)
    t = torch.tensor([dev_ms], dtype=torch.float64, device=tdev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    clocks = clk.summary()

    # End to end through the C-ABI with host buffers: program text -> parse ->
    # device tables (H2D) -> simulate -> norm + 2^20-amplitude window (D2H).
    window = 1 << 20
    host = torch.empty(window * 2, dtype=torch.float64).pin_memory().numpy().view(np.complex128)
    e2e = []
    for _ in range(max(1, min(args.steps, 3))):
        barrier()
        t1 = time.perf_counter()
        p2 = qk.Program.parse(prog_text, cfg)
        st.simulate(p2, 0)
        nrm = st.norm()
        st.download(0, window, out=host)
        barrier()
        e2e.append(time.perf_counter() - t1)
        del p2
    e2e_s = sorted(e2e)[len(e2e) // 2]
    if world > 1:  # the norm of the whole state: sum of the slices' sum |a|^2
        nt = torch.tensor([nrm], dtype=torch.float64, device=tdev)
        dist.all_reduce(nt, op=dist.ReduceOp.SUM)
        nrm = float(nt.item())
    et = torch.tensor([e2e_s, cold_s], dtype=torch.float64, device=tdev)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_s, cold_s = float(et[0].item()), float(et[1].item())

    # Roofline of the dominant kernel, the fused block pass over the whole
    # slice: algorithmic bytes per launch (32 B/amplitude,
    # read + write) over its event-timed average launch.  Passes of a run from
    # a basis state that still have known zeros in their input ("sparse")
    # write every amplitude but read only the support: their algorithmic
    # bytes are 16 B/amp + 16 B per amplitude not known to be zero.  The first
    # pass of a run (the one tile holding |initial>) is reported apart as init.
    amps = 1 << (n - R)
    peak, peak_src = measured_peaks()
    fp_launches = sum(x["full_pass_launches"] for x in stats)
    fp_ms = sum(x["full_pass_ms"] for x in stats)
    fp_bytes = sum(x["full_pass_bytes"] for x in stats)
    sp_launches = sum(x["sparse_pass_launches"] for x in stats)
    sp_ms = sum(x["sparse_pass_ms"] for x in stats)
    sp_bytes = sum(x["sparse_pass_bytes"] for x in stats)
    launches = fp_launches + sp_launches
    pass_launch_ms = (fp_ms + sp_ms) / max(1, launches)
    pass_bytes_per_launch = (fp_bytes + sp_bytes) / max(1, launches)
    pass_gbs = pass_bytes_per_launch / (pass_launch_ms * 1e-3) / 1e9 if launches else 0.0
    s0 = stats[-1]
    tr = ncu_traffic()
    # ncu DRAM bytes per amplitude of each pass kind (profiles/block_pass_traffic.json,
    # from an ncu --set full capture of the same program family at 31 qubits),
    # scaled to this slice and averaged over this step's launches like `achieved`
    by_kind = (tr or {}).get("dram_bytes_per_amp_by_kind", {})
    traffic = round((by_kind["full"] * fp_launches + by_kind["sparse"] * sp_launches) / launches * amps) \
        if launches and "full" in by_kind and "sparse" in by_kind else None
    # program-level roofline: T_roof = sum over items, HBM-bound
    t_roof = (s0["block_bytes"] + s0["ims_bytes"]) / (peak * 1e9) + s0["xrs_bytes"] / 900e9

    out = {
        "metric": METRIC,
        "value": round(ms_per_step / 1e3, 6),
        "unit": "s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 3),
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "c128 (fp64 complex)",
        "data": "synthetic: generated circuit, |0> initial state",
        "config": {"workload": f"{kind.upper()}-{n} ({kind}, {n} qubits, {1 << R} GPU(s), 2^{n - R} amps/GPU)",
                   "n_qubits": n, "rank_qubits": R, "chunk_qubits": args.chunk, "fusion": 0,
                   "xrs": (transport + (" (grouped ncclSend/ncclRecv, 2^B receive buffer, copy-back)"
                                        if transport == "nccl" else " (cudaIpc-mapped peer slices, in-place swap)"))
                   if world > 1 else None,
                   "diagonal_fusion": 0, "program": counts, "optimize_s": round(opt_s, 3),
                   "l2": f"state {16 * amps / 2**30:.0f} GiB/GPU >> 126 MB L2: inputs larger than L2, no flush"},
        "e2e": {"value": round(e2e_s, 6), "unit": "s", "h2d_bytes_per_step": len(prog_text.encode()),
                "d2h_bytes_per_step": window * 16 + 8,
                "path": "qk_program_parse + qk_simulate + qk_norm + qk_download(2^20 amps) via C-ABI; the "
                        "re-parsed program hits the process-wide schedule cache (compiled + autotuned schedule "
                        "reused)",
                "cold_first_call_s": round(cold_s, 3),
                "cold_note": "first qk_simulate of the program in this process: NVRTC specialization of every "
                             "pass variant (disk cache empty on a fresh box), table upload, first autotune run"},
        "gpu_launches": int(sum(x["kernel_launches"] for x in stats)),
        "roofline": {"bound": "hbm", "kernel": "qk_pass_<hash> (NVRTC-specialized fused pass over the whole "
                                               "slice, csrc/engine/jit.cpp)",
                     "achieved": round(pass_gbs, 1),
                     "peak": peak, "unit": "GB/s", "frac": round(pass_gbs / peak, 4),
                     "peak_source": peak_src, "traffic": traffic,
                     "traffic_source": (tr["source"] + "; DRAM bytes/amp per pass kind x this slice") if traffic else None,
                     "algorithmic_bytes_per_launch": round(pass_bytes_per_launch),
                     "launches_per_step": launches // max(1, args.steps),
                     "avg_launch_ms": round(pass_launch_ms, 3),
                     "passes_per_step": {
                         "full": {"launches": fp_launches // max(1, args.steps),
                                  "ms": round(fp_ms / args.steps, 3),
                                  "gbs": round(fp_bytes / max(1e-9, fp_ms * 1e-3) / 1e9, 1) if fp_ms else None},
                         "sparse": {"launches": sp_launches // max(1, args.steps),
                                    "ms": round(sp_ms / args.steps, 3),
                                    "algorithmic_bytes": round(sp_bytes / args.steps),
                                    "gbs": round(sp_bytes / max(1e-9, sp_ms * 1e-3) / 1e9, 1) if sp_ms else None}},
                     "excludes": "the run's first pass (the single tile holding |initial>, no memset: the next pass "
                                 "writes every tile), reported as breakdown.init_ms",
                     "fp64_peak_tflops_measured": 36.5,
                     "fp64_note": "DFMA 36.5 / DMMA 37.0 TF measured (profiles/r1_fp64_peak.txt)"},
        "breakdown": {"block_ms": round(s0["block_ms"], 2), "full_pass_ms": round(s0["full_pass_ms"], 2),
                      "sparse_pass_ms": round(s0["sparse_pass_ms"], 2),
                      "init_ms": round(s0["init_ms"], 2), "ims_ms": round(s0["ims_ms"], 2),
                      "xrs_ms": round(s0["xrs_ms"], 2), "block_launches": s0["block_launches"],
                      "ims_launches": s0["ims_launches"], "xrs_rounds": s0["xrs_rounds"],
                      "ims_gbs": round(s0["ims_bytes"] / max(1e-9, s0["ims_ms"] * 1e-3) / 1e9, 1)
                      if s0["ims_ms"] else None,
                      "xrs_nvlink_gbs_per_direction": round(s0["xrs_bytes"] / max(1e-9, s0["xrs_ms"] * 1e-3) / 1e9, 1)
                      if s0["xrs_ms"] else None,
                      "program_roofline_s": round(t_roof, 4),
                      "program_roofline_frac": round(t_roof / (ms_per_step / 1e3), 4),
                      "autotune_runs": tune_runs,
                      "norm": nrm},
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline(args, kind, n, st, qk)
        except Exception as e:  # noqa: BLE001
            out["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    if rank == 0:
        print(json.dumps(out), flush=True)
    st.close()
    if world > 1:
        dist.destroy_process_group()


def gpu_time_program(qk, kind, n, chunk, reps=5):
    """Device-timed steps (CUDA events inside qk_simulate) of this engine on the
    same program, after its autotune settled; median of `reps`."""
    cfg = qk.Config.make(n, 0, chunk=chunk, fusion=0, diag=0)
    a, seed = circuit_args(kind, n)
    prog = qk.Program.optimize(qk.generate(kind, n, a, seed), cfg)
    st = qk.State(n)
    try:
        for _ in range(24):
            if not st.simulate(prog, 0)["tuning_runs"]:
                break
        ts = sorted(st.simulate(prog, 0)["total_ms"] for _ in range(reps))
        return ts[len(ts) // 2] / 1e3
    finally:
        st.close()


def cpu_baseline(args, kind, n, st, qk):
    """The reference's simulateProgram on this box's host cores: one measured
    run at --cpu-sample-qubits (the same program family: chunk_qbit, fusion
    off), extrapolated to the n-qubit workload by amplitude-passes, plus the
    same-size GPU/CPU pair measured in this run."""
    threads = os.cpu_count() or 1
    ns = min(args.cpu_sample_qubits, n)
    sec, items_s, _ = cpu_reference_run(kind, ns, args.chunk, threads)
    v, scale, items_t = extrapolate(kind, ns, sec, items_s, n, args.chunk)
    gpu_s = gpu_time_program(qk, kind, ns, min(args.chunk, ns))
    return {"value": round(v, 3), "unit": "s", "cores": threads, "kind": "reference",
            "extrapolated": ns != n,
            "sample": f"reference simulateProgram (oracle/_ref, unmodified reference sources) on {kind.upper()}-{ns} "
                      f"(chunk_qbit {min(args.chunk, ns)}, fusion off, {items_s} items), {threads} threads: "
                      f"{sec:.3f} s measured, x{scale:.1f} by amplitude-passes to the {n}-qubit program "
                      f"({items_t} items); a {n}-qubit host state needs {16 * 2**n / 2**30:.0f} GiB",
            "measured_pair": {"workload": f"{kind.upper()}-{ns}, same program, this box",
                              "cpu_s": round(sec, 3), "gpu_s": round(gpu_s, 5),
                              "cpu_over_gpu": round(sec / gpu_s, 1) if gpu_s else None},
            "full_size_check": full_size_reference(kind, n)}


def full_size_reference(kind, n):
    """The one full-size reference run on record (not this run: it takes ~8 min
    and 128 GiB of host RAM; profiles/r2_reference_cpu_full_size.json)."""
    path = os.path.join(ROOT, "profiles", "r2_reference_cpu_full_size.json")
    if not os.path.exists(path):
        return None
    d = json.load(open(path))
    for r in d.get("runs", []):
        if r.get("workload", "").startswith(f"{kind.upper()}-{n} "):
            return {"workload": r["workload"], "cpu_s": r["simulate_s"], "threads": r["threads"],
                    "source": "profiles/r2_reference_cpu_full_size.json (tools/ref_cpu_full.py, gpurun box host)"}
    return None


def run_reference(args, rank, n, R, kind):
    """--impl reference: the reference's own CPU implementation (oracle/_ref =
    /root/reference/proj/src compiled unmodified) on the host cores, rank 0
    only.  This process never loads libqk_b200.so.  Each step is a bounded
    sample: simulateProgram at --ref-sample-qubits, extrapolated to n qubits
    by amplitude-passes (the whole --steps/--warmup run stays within minutes)."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    ns = min(args.ref_sample_qubits, n)
    vals, secs = [], []
    items_s = None
    for i in range(args.warmup + args.steps):
        warm = i < args.warmup
        sec, items, _ = cpu_reference_run(kind, min(20, ns) if warm else ns, args.chunk, threads)
        if not warm:
            secs.append(sec)
            items_s = items
    sec = sorted(secs)[len(secs) // 2]
    v, scale, items_t = extrapolate(kind, ns, sec, items_s, n, args.chunk)
    vals = [x * scale for x in secs]
    v = sum(vals) / len(vals)
    out = {
        "impl": "reference",
        "metric": METRIC, "value": round(v, 3), "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(v * 1e3, 1), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128 (fp64 complex)",
        "data": "synthetic: generated circuit, |0> initial state",
        "config": {"workload": f"{kind.upper()}-{n} ({kind}, {n} qubits, {1 << R} GPU(s) equivalent)",
                   "n_qubits": n, "chunk_qubits": args.chunk, "fusion": 0, "diagonal_fusion": 0},
        "cpu_baseline": {"value": round(v, 3), "unit": "s", "cores": threads, "kind": "reference",
                         "extrapolated": ns != n,
                         "sample": f"each step: reference simulateProgram on {kind.upper()}-{ns} ({items_s} items, "
                                   f"median {sec:.3f} s measured) x{scale:.1f} amplitude-pass scale to {n} qubits "
                                   f"({items_t} items); warm-up steps run {kind.upper()}-{min(20, ns)}"},
        "e2e": {"value": round(v, 3), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
