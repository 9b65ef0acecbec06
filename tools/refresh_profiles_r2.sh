#!/bin/bash
# Copy the judged summaries of one round-2 GPU batch (tools/probe/gpu_r2z.sh) into profiles/.
# Usage: bash tools/refresh_profiles_r2.sh TAG   (reads gpurun_out/TAG)
set -e
TAG=${1:?tag}
O=gpurun_out/$TAG
C=$(git log -1 --format=%s | cut -c1-80)
tail -1 $O/bench.json > profiles/r2_bench_qft33.json
tail -1 $O/bench_ref.json > profiles/r2_bench_reference_arm.json
cp $O/launches.csv profiles/r2_bench_qft33_launches.csv
{
  echo "# ncu launch list of: python bench.py --steps 2 --warmup 1 --no-cpu-baseline (QFT-33, 1 B200), commit '$C'"
  echo "# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare shares, not absolutes)"
  echo "# (includes the autotune runs before the warm-up: every variant of every pass runs twice)"
  python tools/launch_summary.py $O/launches.csv
  echo
  echo "# steady state: the last step's launches"
  python tools/launch_tail.py $O/launches.csv 6 2>/dev/null || true
} > profiles/r2_bench_qft33_launches.txt
{
  echo "# ncu --set full --clock-control none of QFT-31 (tools/run_qft.py 31): the passes after the basis tile, commit '$C'"
  echo "# support-aware DP (work weight 250), tight support, Toffoli fusion, CTA-bit controls, deferred H scales; the last (filling) pass reads the support and writes every tile (staged TMA stores)"
  python tools/ncu_summary.py $O/prof_qft31.ncu-rep --sass
} > profiles/r2_qft31_sparse_dp_ncu_full.txt
{
  echo "# per-pass device times after autotune at 33 qubits (tools/family_passes.py KIND 33), commit '$C'"
  for k in qft bvones qaoa random grover; do echo "## $k"; grep -v "^----" $O/fam_$k.txt; grep -v "^----\|^$" $O/fam_$k.err | head -40; done
} > profiles/r2_families33_passes.txt
[ -f $O/summary_grover.txt ] && { echo "# ncu --set full of Grover-31 (QK_TUNE=0, primary variants), Toffoli fusion + CTA controls; commit '$C'"; cat $O/summary_grover.txt; } > profiles/r2_grover31_ncu_full.txt
python - "$O" <<'PY'
import csv, io, json, subprocess, sys
rep = sys.argv[1] + "/prof_qft31.ncu-rep"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
rd, wr = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
per = [round(float(r[rd].replace(",", "")) * scale[u[rd]] + float(r[wr].replace(",", "")) * scale[u[wr]]) for r in rows[2:]]
path = "profiles/block_pass_traffic.json"
d = json.load(open(path))
d["per_launch_measured"]["qft31_sparse"] = per
d["dram_bytes_per_amp_by_kind"]["sparse"] = round(sum(per) / len(per) / (1 << 31), 3)
d["source"] = ("profiles/r2_qft31_sparse_dp_ncu_full.txt (QFT-31 passes 2-3 after the support-aware DP: deferred zeros + "
               "sparse reads, staged TMA stores) and profiles/r2_qft31_random31_ncu_full.txt (random-31 passes 10-11, full)")
json.dump(d, open(path, "w"), indent=2)
print(json.dumps(d["dram_bytes_per_amp_by_kind"]))
PY
