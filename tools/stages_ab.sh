# A/B of the in-tree build against ab/ builds on the main layer shapes
libs=${1:-"default base"}
for rep in 1 2; do
  for wl in c2:0 c2a:0 c3:0; do
    for l in $libs; do
      if [ "$l" = default ]; then unset LKG_LIB; else export LKG_LIB=$PWD/ab/liblutkan_$l.so; fi
      echo -n "[$l] "; timeout 300 python tools/time_layer.py ${wl%%:*} ${wl##*:} 50 2>&1 | tail -1
    done
  done
done
for l in $libs; do
  if [ "$l" = default ]; then unset LKG_LIB; else export LKG_LIB=$PWD/ab/liblutkan_$l.so; fi
  echo -n "[$l] "; timeout 300 python tools/time_layer.py c4 1 3 2>&1 | tail -1
done
