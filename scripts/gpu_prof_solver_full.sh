#!/bin/bash
# ncu --set full of one whole C4 deflated iteration (11 kernels, warm): the regex skips the probing matvecs of
# prepare(); 344 matching launches precede the first iteration (restrictions / prolongations of the coarse assembly)
mkdir -p gpurun_out
python scripts/prof_solve.py 160 80 80 8 8 > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --cache-control none --import-source on \
    -k regex:"k_matvec<256, 2, [01], 1|k_pcg_update|k_restrict|k_coarse|k_top|k_block_nu|k_prolong" -s 388 -c 11 -f \
    -o gpurun_out/c4_iter_full python scripts/prof_solve.py 160 80 80 8 8 > gpurun_out/ncu_c4_full.log 2>&1
echo "ncu c4 full $?"
ncu -i gpurun_out/c4_iter_full.ncu-rep --page raw --csv > gpurun_out/c4_iter_full_raw.csv 2>/dev/null
