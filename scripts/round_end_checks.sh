# GPU box: full GPU tests, reference arm, bench, and ncu evidence (launch list of one cfg2 step;
# --set full of the CGS2 step kernels on the workload shape; the filter and KPM kernels)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
python bench.py --steps 2 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rw_stream -c 3 -o gpurun_out/r2_rw_cgs2_k1440 python scripts/cgs2_bench.py "262144,1440" > gpurun_out/ncu_rw.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_rw.log
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r2_launches_cfg2.csv python scripts/run_cfg.py cfg2 --jobs 1 --only 7 > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
