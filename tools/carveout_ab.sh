# A/B the shared-memory carveout hook on one layer: bash tools/carveout_ab.sh <workload> <layer> <iters> [values...]
wl=$1; layer=$2; it=$3; shift 3
echo -n "[carveout default] "; timeout 600 python tools/time_layer.py $wl $layer $it 2>&1 | tail -1
for v in "$@"; do
  echo -n "[carveout $v] "; LKG_CARVEOUT=$v timeout 600 python tools/time_layer.py $wl $layer $it 2>&1 | tail -1
done
