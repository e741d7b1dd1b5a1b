set -x
NCU=/usr/local/cuda/bin/ncu
timeout 600 python -m pytest tests/test_gpu_bicgstab.py -q > gpurun_out/bicg3.log 2>&1; tail -1 gpurun_out/bicg3.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2d.log 2>&1; tail -1 gpurun_out/bench_c2d.log
CFG=c2 KMAX=8 SOLVER=bicgstab $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_bi_ -c 400 --csv --log-file gpurun_out/p_bicg_launches2.csv python tools/prof_c3.py > gpurun_out/p_bicg_ncu2.log 2>&1
python tools/prof_c2.py > gpurun_out/p_c2_plain.log 2>&1 && \
$NCU --set full --clock-control none --import-source on -k regex:k_gmres_persistent -s 60 -c 1 -o gpurun_out/prof_c2_full python tools/prof_c2.py > gpurun_out/p_c2_ncu.log 2>&1
