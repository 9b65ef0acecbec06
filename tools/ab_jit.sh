for cfg in "1 1" "1 0" "0 0"; do set -- $cfg
  QK_JIT_PERSIST=$1 QK_JIT_PF=$2 TAG="P$1F$2" timeout 600 python tools/blockbench.py 32 13 2>&1 | tail -16
done
QK_JIT_MIN_QUBITS=-1 TAG=interp timeout 600 python tools/blockbench.py 32 13 2>&1 | tail -1
