# round 2: closing validation -- full GPU suite (default and plan forced), smoke, bench (both arms),
# config-3 line, launch list and ncu captures of the headline kernel and the persistent kernel
set -x
O=gpurun_out/closing
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
SAD_SPMM_BAND=1 timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu_bandforced.log 2>&1; tail -3 $O/pytest_gpu_bandforced.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -8 $O/smoke.log
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 400 $O/bench_ref.json
timeout 1200 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; tail -c 600 $O/bench_c4.json; tail -3 $O/bench_c4.err
timeout 1200 python bench.py --config c3 --no-cpu-baseline --steps 1 --warmup 1 > $O/bench_c3.json 2> $O/bench_c3.err; tail -c 300 $O/bench_c3.json
timeout 600 python bench.py --config c2 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 300 $O/bench_c2.json
timeout 900 python bench.py --rowpart --no-cpu-baseline --steps 5 > $O/bench_c4_rowpart.json 2> $O/bench_c4_rowpart.err; tail -c 300 $O/bench_c4_rowpart.json
timeout 2400 python bench.py --config c5 --no-cpu-baseline --steps 1 --warmup 1 > $O/bench_c5.json 2> $O/bench_c5.err; tail -c 300 $O/bench_c5.json
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_c4.csv python bench.py --no-c3 --no-cpu-baseline --steps 5 --warmup 3 --c4-steps 2 > $O/ncu_launch.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmm_band -s 4 -c 1 -o $O/prof_c4_band python bench.py --no-c3 --no-cpu-baseline --steps 3 --warmup 3 --c4-steps 2 > $O/ncu_band.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gmres_persistent -c 2 -o $O/prof_c4_pers python bench.py --no-c3 --no-cpu-baseline --steps 3 --warmup 3 > $O/ncu_pers.log 2>&1
ls -la $O
