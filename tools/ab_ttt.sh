#!/bin/bash
# A/B of the Table-1 time-to-tolerance probe for two builds: tools/ab_ttt.sh <libA.so> <libB.so>
for L in "$1" "$2"; do
  echo "== $L"; BICADMM_LIB_PATH=$L timeout 600 python tools/ttt_probe.py 2>&1 | tail -4
done
