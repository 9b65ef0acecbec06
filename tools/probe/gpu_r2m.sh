O=gpurun_out/r2m; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2m
for k in qft bvones qaoa random grover; do
  timeout 300 python tools/family_passes.py $k 33 > $O/fam_$k.txt 2> $O/fam_$k.err; cat $O/fam_$k.txt | grep -v "^----"; sed -n '/---- tuned run/,$p' $O/fam_$k.err | grep "qk item" | tr '\n' ' ' | cut -c1-300; echo
done
timeout 900 python bench.py --steps 10 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc $?"; cat $O/bench.json | cut -c1-600; tail -3 $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_ncu.log 2>&1; echo "ncu-list rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qk_pass -s 1 -c 2 -o $O/prof_qft31 python tools/run_qft.py 31 > $O/ncu_qft.log 2>&1; echo "ncu qft rc $?"
QK_IMS_TILED=1 timeout 600 python tools/imsbench.py 33 > $O/ims33_tiled.txt 2>&1; cat $O/ims33_tiled.txt
QK_IMS_TILED=0 timeout 600 python tools/imsbench.py 33 > $O/ims33_generic.txt 2>&1; cat $O/ims33_generic.txt
timeout 1700 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $O/pytest_gpu.log
