# ncu --set full of the C4 coarse-solve kernels (leaf forward, top tiles, leaf backward)
mkdir -p gpurun_out
python scripts/prof_solve.py 160 80 80 8 8 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_coarse_fwd|k_top_tiles|k_coarse_bwd" -s 12 -c 3 -o gpurun_out/c4_coarse_full_r01c python scripts/prof_solve.py 160 80 80 8 8 > gpurun_out/ncu_cf.log 2>&1; echo "ncu coarse full $?"
