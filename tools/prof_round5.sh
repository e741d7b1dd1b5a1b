# Round-1 closing measurements: bench lines (c2 headline, c4, c3), the ncu launch
# list of one config-2 solve (all kernels) and the persistent kernel's DRAM traffic.
set -x
NCU=/usr/local/cuda/bin/ncu
python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err
python bench.py --config c4 > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err
python tools/prof_c2.py > gpurun_out/p5_c2_plain.log 2>&1 && \
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p5_c2_launches.csv python tools/prof_c2.py > gpurun_out/p5_c2_ncu_l.log 2>&1
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gmres_persistent -o gpurun_out/p5_c2_traffic python tools/prof_c2.py > gpurun_out/p5_c2_ncu_t.log 2>&1
python bench.py --config c3 --steps 1 --warmup 1 > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err
