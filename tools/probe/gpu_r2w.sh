O=gpurun_out/r2w; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2w
# primary variants only (QK_TUNE=0), one run; summaries kept, reports dropped (size)
for k in grover bvones qaoa; do
  QK_TUNE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:qk_pass -c 20 -o /tmp/prof_${k}31 -f python tools/run_qft.py 31 13 1 $k > $O/ncu_$k.log 2>&1; echo "ncu $k rc $?"
  python tools/ncu_summary.py /tmp/prof_${k}31.ncu-rep --sass > $O/summary_$k.txt 2>&1
done
