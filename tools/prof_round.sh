set -x
NCU=/usr/local/cuda/bin/ncu
python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/c4_plain.log 2>&1 && \
$NCU --set full --clock-control none --import-source on -k regex:k_spmm_bulk -s 3 -c 1 -o gpurun_out/prof_c4_spmm python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/ncu_c4a.log 2>&1
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gmres_persistent -c 2 -o gpurun_out/prof_c4_pers python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/ncu_c4b.log 2>&1
python tools/prof_c2.py > gpurun_out/c2_plain.log 2>&1 && \
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gmres_persistent -o gpurun_out/prof_c2_pers python tools/prof_c2.py > gpurun_out/ncu_c2a.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:k_gmres_persistent -s 60 -c 1 -o gpurun_out/prof_c2_full python tools/prof_c2.py > gpurun_out/ncu_c2b.log 2>&1
ls -la gpurun_out
