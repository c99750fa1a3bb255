mkdir -p gpurun_out
python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/prof4_plain.log 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on -k regex:"k_coarse_fwd|k_coarse_bwd" -s 14 -c 14 -o gpurun_out/coarse_full python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/ncu4.log 2>&1
echo "ncu exit $?"
