O=gpurun_out/r2n; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2n
for k in qft bvones qaoa random grover; do
  timeout 300 python tools/family_passes.py $k 33 > $O/fam_$k.txt 2> $O/fam_$k.err; cat $O/fam_$k.txt | grep -v "^----"; sed -n '/---- tuned run/,$p' $O/fam_$k.err | grep "qk item" | tr '\n' ' ' | cut -c1-200; echo
done
timeout 300 python tools/family_passes.py qft 30 2>/dev/null | grep -v "^----"
timeout 900 python bench.py --steps 10 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc $?"; cat $O/bench.json | cut -c1-400; tail -3 $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 2 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc $?"; cat $O/bench_ref.json | cut -c1-300
timeout 1700 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?"; tail -3 $O/smoke.log
