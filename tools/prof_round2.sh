set -x
NCU=/usr/local/cuda/bin/ncu
python tools/prof_c3.py > gpurun_out/p_c3_plain.log 2>&1 && \
$NCU --set full --clock-control none --import-source on -k regex:k_gmres_persistent -c 1 -o gpurun_out/prof_c3_full python tools/prof_c3.py > gpurun_out/p_c3_ncu.log 2>&1
CFG=c2 KMAX=8 SOLVER=bicgstab python tools/prof_c3.py > gpurun_out/p_bicg_plain.log 2>&1 && \
CFG=c2 KMAX=8 SOLVER=bicgstab $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_bi_ -c 400 --csv --log-file gpurun_out/p_bicg_launches.csv python tools/prof_c3.py > gpurun_out/p_bicg_ncu.log 2>&1
python bench.py --config c4 --rowpart --c4-n0 4096 --c4-steps 30 --steps 1 --warmup 3 > gpurun_out/p_c4rp_plain.log 2>&1 && \
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_dot_dual|k_update|k_spmm|k_dist|k_halo|k_group" -s 20 -c 300 --csv --log-file gpurun_out/p_c4rp_launches.csv python bench.py --config c4 --rowpart --c4-n0 4096 --c4-steps 30 --steps 1 --warmup 3 > gpurun_out/p_c4rp_ncu.log 2>&1
ls -la gpurun_out | tail -20
