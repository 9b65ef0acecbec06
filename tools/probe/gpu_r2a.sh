O=gpurun_out/r2a; mkdir -p $O
{ nproc; free -g; cat /sys/fs/cgroup/memory.max 2>/dev/null; lscpu | grep -i "model name\|^CPU(s)"; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; } > $O/host.txt 2>&1
cat $O/host.txt
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/probe/nccl_same_gpu.py > $O/nccl_probe.log 2>&1; echo "nccl probe rc $?"; grep -i "rank\|error" $O/nccl_probe.log | head -5
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2
timeout 1500 python -m pytest tests/test_gpu_large_parity.py -m gpu -q --durations=20 > $O/pytest_large.log 2>&1; echo "pytest large rc $?"; tail -30 $O/pytest_large.log
timeout 1300 python -m pytest tests -m gpu -q --durations=30 --ignore=tests/test_gpu_large_parity.py > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -40 $O/pytest_gpu.log
