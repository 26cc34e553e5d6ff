# timeline of the tiled kernel under named conv_opts (PC_OPT), per library variant
# usage: bash tools/gpu_tl_opt.sh OUTDIR "opt1;opt2" "v1 v2"
mkdir -p gpurun_out/$1
IFS=';' read -ra OPTS <<< "$2"
for v in $3; do
  i=0
  for o in "${OPTS[@]}"; do
    PC_OPT="$o" PC_LIB_PATH=$PWD/tools/variants/$v.so timeout 300 python tools/tiled_timeline.py cfg2 > gpurun_out/$1/tl_${v}_$i.json 2> gpurun_out/$1/tl_${v}_$i.err
    i=$((i+1))
  done
done
echo done
