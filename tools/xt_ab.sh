# A/B of the XT table walk (transposed input, 2D TMA x blocks) against the row-major path (LKG_XT=0)
for rep in 1 2; do
  for wl in c3:0 c2:0; do
    echo -n "[xt] "; timeout 300 python tools/time_layer.py ${wl%%:*} ${wl##*:} 50 2>&1 | tail -1
    echo -n "[rowmajor] "; LKG_XT=0 timeout 300 python tools/time_layer.py ${wl%%:*} ${wl##*:} 50 2>&1 | tail -1
  done
done
echo -n "[xt] "; timeout 300 python tools/time_layer.py c4 1 3 2>&1 | tail -1
echo -n "[rowmajor] "; LKG_XT=0 timeout 300 python tools/time_layer.py c4 1 3 2>&1 | tail -1
