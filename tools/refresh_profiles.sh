#!/bin/bash
# Copy the judged summaries of one tools/gpu_round.sh run into profiles/.
# Usage: bash tools/refresh_profiles.sh TAG   (reads gpurun_out/TAG)
set -e
TAG=${1:?tag}
O=gpurun_out/$TAG
C=$(git log -1 --format=%s | cut -c1-80)
cp $O/bench.json profiles/r1_bench_qft33.json
cp $O/launches.csv profiles/r1_bench_qft33_launches.csv
{
  echo "# ncu launch list of: python bench.py --steps 1 --warmup 1 --no-cpu-baseline (QFT-33, 1 B200), commit '$C'"
  echo "# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare shares, not absolutes)"
  echo "# (includes the autotune runs before the warm-up: every register-width / tile-size variant runs once)"
  python tools/launch_summary.py $O/launches.csv
} > profiles/r1_bench_qft33_launches.txt
{
  echo "# ncu --set full --clock-control none of QFT-31 (tools/run_qft.py 31): the two full-state fused passes"
  echo "# (launch 0, the synthesized single-tile first pass, is skipped); commit '$C'"
  echo "# algorithmic bytes per launch = 32 B x 2^31 = 68.72 GB"
  python tools/ncu_summary.py $O/prof_block.ncu-rep --sass
} > profiles/r1_qft31_ncu_full.txt
python - "$O" <<'PY'
import csv, io, json, subprocess, sys
rep = sys.argv[1] + "/prof_block.ncu-rep"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
rd, wr = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
per = [round(float(r[rd].replace(",", "")) * scale[u[rd]] + float(r[wr].replace(",", "")) * scale[u[wr]]) for r in rows[2:]]
amps = 1 << 31
json.dump({
    "kernel": "qk_pass_<hash> (specialized fused block pass)",
    "source": "profiles/r1_qft31_ncu_full.txt: ncu --set full, QFT-31, the 2 full-state passes",
    "dram_bytes_per_launch_measured": per,
    "algorithmic_bytes_per_launch": 32 * amps,
    "dram_bytes_per_amp": round(sum(per) / len(per) / amps, 3),
    "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch at 2^31 amplitudes; the pass reads and "
            "writes each amplitude once.  bench.py scales bytes/amp to its slice."},
    open("profiles/block_pass_traffic.json", "w"), indent=2)
print(open("profiles/block_pass_traffic.json").read())
PY
