# A/B: nu = S mu inside the prolongation (new lib) vs k_block_nu + prolongation (old lib); batch + parity on the new one
mkdir -p gpurun_out
L=paper_2203_15115_b200/libtopovox_b200.so
for rep in 1 2; do for v in old new; do
  cp ab_$v.so $L
  echo "$v C4 $(timeout 900 python scripts/iter_bench.py 160 80 80 8 300 2>&1 | tail -1 | cut -c40-75)  C3 $(timeout 900 python scripts/iter_bench.py 80 40 40 4 200 2>&1 | tail -1 | cut -c40-75)  C5 $(timeout 900 python scripts/iter_bench.py 320 160 160 8 60 2>&1 | tail -1 | cut -c40-75)"
done; done
for v in old new; do cp ab_$v.so $L; echo "$v batch $(timeout 900 python scripts/batch_bench.py 2>&1 | tail -2 | tr '\n' ' ' | cut -c150-300)"; done
cp ab_new.so $L
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
