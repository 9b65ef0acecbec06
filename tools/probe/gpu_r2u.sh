O=gpurun_out/r2u; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2u
for k in qft bvones qaoa random grover; do
  timeout 600 python tools/family_passes.py $k 33 > $O/fam_$k.txt 2> $O/fam_$k.err; grep -v "^----" $O/fam_$k.txt
done
timeout 300 python tools/family_passes.py qft 30 2>/dev/null | grep -v "^----"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_ncu.log 2>&1; echo "ncu-list rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qk_pass -s 1 -c 2 -o $O/prof_qft31 python tools/run_qft.py 31 > $O/ncu_qft.log 2>&1; echo "ncu qft rc $?"
