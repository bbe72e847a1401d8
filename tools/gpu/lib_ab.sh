# A/B of library builds: LIBS="default w12r3" CASES="c2:0 c3:0" bash tools/gpu/lib_ab.sh
for c in ${CASES:-c2:0 c2a:0 c3:0 c4:1}; do
  wl=${c%%:*}; layer=${c##*:}; it=50; [ $wl = c4 ] && it=5
  for l in ${LIBS:-default}; do
    if [ "$l" = default ]; then unset LKG_LIB; else export LKG_LIB=$PWD/ab/liblutkan_$l.so; fi
    echo -n "[$l] "; timeout 300 python tools/time_layer.py $wl $layer $it 2>&1 | tail -1
  done
done
