# GPU box: parity tests, the CGS2 step microbenchmark and a short cfg2 bench (evidence run)
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python scripts/cgs2_bench.py "262144,100;262144,400;262144,1000;262144,1440;262144,2880;2097152,1000;2097152,4000" > gpurun_out/cgs2_bench.log 2>&1
python bench.py --steps 1 --warmup 2 --no-cpu --no-others --no-e2e > gpurun_out/bench_quick.log 2>&1
