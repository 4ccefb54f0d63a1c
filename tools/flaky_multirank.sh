#!/bin/bash
# Repeat the loopback multi-rank tests under different stream settings and count failures.
cd "$(dirname "$0")/.."
for mode in ${MODES:-default VB_NO_PDL VB_NO_PRIO}; do
  fails=0
  for i in $(seq 1 ${1:-6}); do
    if [ "$mode" = default ]; then env=""; else case "$mode" in *=*) env="$mode";; *) env="$mode=1";; esac; fi
    out=$(env $env timeout 200 python -m pytest tests/test_gpu_multirank.py -q -x -k "irregular or rank_grid0 or rank_grid1" 2>&1)
    if echo "$out" | tail -1 | grep -q failed; then
      fails=$((fails+1))
      echo "$mode run $i: $(echo "$out" | grep -E '^E .*rank errors|FAILED' | head -2 | cut -c1-400)"
    fi
  done
  echo "$mode: $fails failures"
done
