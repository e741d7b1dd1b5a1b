timeout 600 python tools/spmm_band_probe.py c3 2>&1 | grep "GB/s"
timeout 600 python tools/spmm_band_probe.py c3 4 2>&1 | grep "GB/s"
