for l in default xb1; do
  if [ "$l" = default ]; then unset LKG_LIB; else export LKG_LIB=$PWD/ab/liblutkan_$l.so; fi
  echo -n "[$l] "; timeout 300 python tools/time_layer.py c4 1 3 2>&1 | tail -1
  echo -n "[$l] "; timeout 600 python tools/time_layer.py c5 0 3 2>&1 | tail -1
  echo -n "[$l] "; timeout 300 python tools/time_layer.py c3 0 50 128 2>&1 | tail -1
  echo -n "[$l] "; timeout 300 python tools/time_layer.py c3 0 50 16 2>&1 | tail -1
done
