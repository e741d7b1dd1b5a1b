set -x
O=gpurun_out/r2c
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmm_band -s 4 -c 1 -o $O/prof_c4_band python bench.py --no-c3 --no-cpu-baseline --steps 3 --warmup 3 --c4-steps 2 > $O/ncu_band.log 2>&1
tail -3 $O/ncu_band.log
