# SpMM x-window staging sweep of the tuning harness (config-4 operator)
mkdir -p gpurun_out/r2
for b in tools/bin_spmm_*; do for xw in 0 2 3 4; do ./$b 4096 $xw; done; done > gpurun_out/r2/spmm_sweep4.txt 2>&1
cat gpurun_out/r2/spmm_sweep4.txt
