# A/B: in-tree build vs ab/liblutkan_xb1.so (one x buffer) with and without a carveout hint
for rep in 1 2; do for wl in c2:0 c2a:0 c3:0; do
  unset LKG_LIB LKG_CARVEOUT
  echo -n "[default] "; timeout 300 python tools/time_layer.py ${wl%%:*} ${wl##*:} 50 2>&1 | tail -1
  export LKG_LIB=$PWD/ab/liblutkan_xb1.so
  echo -n "[xb1] "; timeout 300 python tools/time_layer.py ${wl%%:*} ${wl##*:} 50 2>&1 | tail -1
  export LKG_CARVEOUT=50
  echo -n "[xb1 co50] "; timeout 300 python tools/time_layer.py ${wl%%:*} ${wl##*:} 50 2>&1 | tail -1
done; done
