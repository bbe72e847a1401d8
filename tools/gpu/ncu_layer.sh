# usage: bash tools/gpu/ncu_layer.sh <workload> <layer> <tag>   (one fwd_tiled launch, --set full)
wl=$1; layer=$2; tag=$3
ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-fwd_tiled} -c 1 -f -o gpurun_out/ncu_$tag \
    python ${PROF:-tools/prof_forward.py} $wl $layer 2 > gpurun_out/ncu_$tag.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_$tag.ncu-rep "$wl layer $layer ($tag)" > gpurun_out/ncu_$tag.txt 2>&1
ncu -i gpurun_out/ncu_$tag.ncu-rep --page raw --csv > gpurun_out/ncu_${tag}_raw.csv 2>/dev/null
[ -n "$SRC" ] && ncu -i gpurun_out/ncu_$tag.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/ncu_${tag}_sass.csv.gz
[ -n "$KEEP_REP" ] || rm -f gpurun_out/ncu_$tag.ncu-rep
