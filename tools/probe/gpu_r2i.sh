O=gpurun_out/r2i; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2i
for k in qft bvones qaoa random grover; do
  timeout 300 python tools/family_passes.py $k 33 > $O/fam_$k.txt 2> $O/fam_$k.err; cat $O/fam_$k.txt | grep -v "^----"; sed -n '/---- tuned run/,$p' $O/fam_$k.err | grep "qk item" | tr '\n' ' ' | cut -c1-400; echo
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_ncu.log 2>&1; echo "ncu-list rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qk_pass -s 1 -c 2 -o $O/prof_qft31 python tools/run_qft.py 31 > $O/ncu_qft.log 2>&1; echo "ncu qft rc $?"; tail -2 $O/ncu_qft.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qk_pass -s 9 -c 2 -o $O/prof_random31 python tools/run_qft.py 31 13 1 random > $O/ncu_random.log 2>&1; echo "ncu random rc $?"; tail -2 $O/ncu_random.log
