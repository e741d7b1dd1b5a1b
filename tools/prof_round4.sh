set -x
NCU=/usr/local/cuda/bin/ncu
python bench.py > gpurun_out/bench_final_c2.log 2> gpurun_out/bench_final_c2.err; tail -1 gpurun_out/bench_final_c2.log
python tools/prof_c2.py > gpurun_out/p_c2_plain2.log 2>&1 && \
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gmres_persistent --csv --log-file gpurun_out/p_c2_launches2.csv python tools/prof_c2.py > gpurun_out/p_c2_ncu_l.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:k_gmres_persistent -s 60 -c 1 -o gpurun_out/prof_c2_full2 python tools/prof_c2.py > gpurun_out/p_c2_ncu2.log 2>&1
python bench.py --gpus 1 --steps 5 --warmup 3 --config c4 > gpurun_out/bench_final_c4.log 2>&1; tail -1 gpurun_out/bench_final_c4.log
