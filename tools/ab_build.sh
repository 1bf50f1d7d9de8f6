#!/bin/bash
# A/B variant of the library: recompile the given sources with extra -D flags
# and link against the in-tree objects.  usage: tools/ab_build.sh NAME "FLAGS" src.cu [src.cu ...]
set -e
name=$1; flags=$2; shift 2
C=/root/repo/paper_1905_05107_b200/csrc
out=/root/repo/abuild/$name; mkdir -p $out
objs=""
for o in $C/*.o; do
  b=$(basename $o .o)
  hit=0; for s in "$@"; do [ "$b.cu" = "$s" ] && hit=1; done
  if [ $hit = 1 ]; then
    nvcc -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v -gencode arch=compute_100a,code=sm_100a $flags -c $C/$b.cu -o $out/$b.o 2> $out/$b.ptxas.log || (cat $out/$b.ptxas.log; exit 1)
    objs="$objs $out/$b.o"
  else objs="$objs $o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libpodsketch_b200.so $objs -lcudart
echo built $out
