set -x
O=gpurun_out/r2e
mkdir -p $O
run() { CFG=c3 KMAX=4 CONC=0 PHASE=tma timeout 600 python tools/c2_phase.py 2>&1 | tail -2 | sed "s/^/PH $1 /"; }
SAD_SPMM_BAND=0 run noband
run band
SAD_GSMEM_KB=60 run band_g60
SAD_GSMEM_KB=60 SAD_SPMM_BAND=0 run noband_g60
SAD_LIB_PATH=$PWD/tools/bin_old.so SAD_SPMM_BAND=0 run old
