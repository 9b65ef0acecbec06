O=gpurun_out/r2q; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2q
for k in qft bvones qaoa random grover; do
  timeout 300 python tools/family_passes.py $k 33 > $O/fam_$k.txt 2> $O/fam_$k.err; grep -v "^----" $O/fam_$k.txt
done
timeout 300 python tools/family_passes.py qft 30 2>/dev/null | grep -v "^----"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc $?"; cut -c1-300 $O/bench.json; tail -3 $O/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc $?"; cut -c1-300 $O/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_ncu.log 2>&1; echo "ncu-list rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qk_pass -s 1 -c 2 -o $O/prof_qft31 python tools/run_qft.py 31 > $O/ncu_qft.log 2>&1; echo "ncu qft rc $?"
timeout 1700 python -m pytest tests -m gpu -q --durations=12 > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -16 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?"; tail -2 $O/smoke.log
