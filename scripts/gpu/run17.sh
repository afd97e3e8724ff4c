python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
mkdir -p gpurun_out/r17
python scripts/prof_tall.py 3 64 64
for a in "3 64 64" "0 128 64" "1 64 64"; do set -- $a
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gram_tc3|update_tc2" -s 1 -c 1 -o gpurun_out/r17/tall_$1_$2 python scripts/prof_tall.py $1 $2 $3 > gpurun_out/r17/ncu_$1_$2.log 2>&1
tail -2 gpurun_out/r17/ncu_$1_$2.log
done
