python scripts/kpm_bench.py 160,160,160 300 128 > gpurun_out/kpm128.log 2>&1
SE_KPM_TRACE=1 python scripts/kpm_bench.py 160,160,160 300 128 >> gpurun_out/kpm128.log 2>&1
