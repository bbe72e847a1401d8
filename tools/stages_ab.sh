# A/B of the in-tree build against ab/liblutkan_base.so on the main layer shapes
for rep in 1 2; do
  for wl in c2:0 c3:0 c2a:0; do
    echo -n "[default] "; timeout 300 python tools/time_layer.py ${wl%%:*} ${wl##*:} 50 2>&1 | tail -1
    echo -n "[base] "; LKG_LIB=$PWD/ab/liblutkan_base.so timeout 300 python tools/time_layer.py ${wl%%:*} ${wl##*:} 50 2>&1 | tail -1
  done
done
echo -n "[default] "; timeout 300 python tools/time_layer.py c4 1 3 2>&1 | tail -1
echo -n "[base] "; LKG_LIB=$PWD/ab/liblutkan_base.so timeout 300 python tools/time_layer.py c4 1 3 2>&1 | tail -1
