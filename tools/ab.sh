#!/bin/bash
# A/B kernel timing: tools/ab.sh "lib1 lib2 ..." "wl:layer wl:layer ..."  (lib "default" = in-tree build)
# Each (workload, layer) is timed with every library, interleaved, twice.
libs=$1; cases=$2; iters=${3:-50}
for rep in 1 2; do
  for c in $cases; do
    wl=${c%%:*}; layer=${c##*:}
    for l in $libs; do
      if [ "$l" = default ]; then unset LKG_LIB; else export LKG_LIB=$PWD/ab/liblutkan_$l.so; fi
      echo -n "[$l] "; timeout 300 python tools/time_layer.py $wl $layer $iters 2>&1 | tail -1
    done
  done
done
