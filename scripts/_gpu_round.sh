python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py --steps 2 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
ncu --set full --import-source on --clock-control none -k regex:k_kpm_ell -s 5 -c 1 -o gpurun_out/kpm_ell -f python scripts/kpm_bench.py 160,160,160 40 16 > gpurun_out/ncu_kpm.log 2>&1
