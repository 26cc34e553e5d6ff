# Source-level stall profile of the headline kernel (ncu --set full + source page, read on the box).
mkdir -p gpurun_out/r02ks
P=gpurun_out/r02ks
C2A="python bench.py --no-sub --no-cpu-baseline --steps 3 --warmup 3 --points asym2_10b"
$C2A > $P/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:pc_tiled_kernel -s 3 -c 1 -o $P/prof $C2A > $P/ncu.log 2>&1
ncu -i $P/prof.ncu-rep --page source --csv --print-source cuda,sass > $P/source.csv 2> $P/source.err
python tools/ncu_source_lines.py $P/source.csv 60 > $P/source_lines.txt 2>&1
ncu -i $P/prof.ncu-rep --page source --csv --print-source sass > $P/sass.csv 2>> $P/source.err
gzip -f $P/source.csv $P/sass.csv
rm -f $P/prof.ncu-rep
echo done
