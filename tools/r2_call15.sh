set -x
O=gpurun_out/r2e
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.mem,clocks.max.mem,power.limit,temperature.gpu --format=csv
for v in old new old new; do
  unset SAD_LIB_PATH
  [ $v = old ] && export SAD_LIB_PATH=$PWD/tools/bin_old.so
  SAD_SPMM_BAND=0 CFG=c3 KMAX=4 CONC=0 PHASE=tma timeout 600 python tools/c2_phase.py 2>&1 | tail -2 | sed "s/^/PH $v /"
done
