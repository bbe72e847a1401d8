# A/B of the table-walk variants (LKG_IDP=0 fp32 lerp, 2 standard lines, default) + a parity subset
for c in ${CASES:-c2:0 c2a:0 c3:0 c4:1}; do
  wl=${c%%:*}; layer=${c##*:}; it=50; [ $wl = c4 ] && it=5
  for v in ${VARIANTS:-0 2 default}; do
    if [ $v = default ]; then unset LKG_IDP; else export LKG_IDP=$v; fi
    echo -n "[IDP=$v] "; timeout 300 python tools/time_layer.py $wl $layer $it 2>&1 | tail -1
  done
done
unset LKG_IDP
[ -n "$NOTEST" ] || python -m pytest tests/test_gpu_parity.py -q -x -k "${TESTS:-layers_c1_c2 or c3_cells or fuzz_compile or c4_layer_rows or c5 or balanced or transposed or tiles_only}" 2>&1 | tail -3
