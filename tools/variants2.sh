export QK_JIT_MIN_QUBITS=0
for cfg in "13 13" "13 12" "12 12" "12 11" "13 11"; do
  set -- $cfg
  echo "== tile $1 chunk $2"
  QK_MAX_TILE_BITS=$1 python tools/profile_items.py 30 $2 | grep -E "total"
done
H13=$(python3 -c "print(';'.join(f'H {q} {q}' for q in range(13)))")
H12=$(python3 -c "print(';'.join(f'H {q} {q}' for q in range(12)))")
QK_MAX_TILE_BITS=12 python tools/passbench.py 30
