set -x
for c in c2:0 c2a:0 c3:0 c4:1; do
  wl=${c%%:*}; layer=${c##*:}; it=50; [ $wl = c4 ] && it=5
  LKG_IDP=0 timeout 300 python tools/time_layer.py $wl $layer $it 2>&1 | tail -1
  timeout 300 python tools/time_layer.py $wl $layer $it 2>&1 | tail -1
done
python -m pytest tests/test_gpu_parity.py -q -x -k "layers_c1_c2 or c3_cells or fuzz_compile or c4_layer_rows or c5 or balanced or transposed or tiles_only" 2>&1 | tail -5
