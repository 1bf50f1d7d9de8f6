#!/bin/bash
# time the config-3 NN shapes on the in-tree build and each abuild/ variant
for v in base "$@"; do
  if [ $v = base ]; then unset POD_LIB_PATH; else export POD_LIB_PATH=$PWD/abuild/$v/libpodsketch_b200.so; fi
  echo "== $v"; python tools/nn3_bench.py
done
