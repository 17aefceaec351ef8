# GPU box: full GPU tests, both bench arms, and the ncu evidence of round 2 (each ncu run only
# after the same command has exited 0 without it)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
python bench.py --steps 2 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
# launch list of one whole slice solve (slice 7 of cfg2: every kernel of the path, graph nodes included)
python scripts/run_cfg.py cfg2 --jobs 1 --only 7 > gpurun_out/run_slice7.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60000 --csv --log-file gpurun_out/r2_launches_cfg2_slice7.csv python scripts/run_cfg.py cfg2 --jobs 1 --only 7 > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
# --set full: the resident filter, the block filter, the DMMA contraction, the CGS2 stream
python scripts/filter_bench.py "64,64,64" 3 > gpurun_out/filter_bench.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cheb_resident -c 2 -o gpurun_out/r2_resident_64 python scripts/filter_bench.py "64,64,64" 3 > gpurun_out/ncu_res.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_res.log
python scripts/filter_bench.py "100,100;40,40,40" 20 > gpurun_out/filter_bench_small.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cheb_resident_ell -c 2 -o gpurun_out/r2_resident_ell_40 python scripts/filter_bench.py "40,40,40" 3 > gpurun_out/ncu_res_ell.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_res_ell.log
python scripts/filter_bench.py "64,64,64;100,100;40,40,40" 20 0 > gpurun_out/filter_bench_perdegree.log 2>&1
python scripts/multi_bench.py "160,160,160" > gpurun_out/multi_bench.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cheb_ell_block -s 10 -c 2 -o gpurun_out/r2_block160 python scripts/multi_bench.py "160,160,160" > gpurun_out/ncu_blk.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_blk.log
python scripts/gemm_bench.py > gpurun_out/gemm_bench.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ritz_gemm -c 2 -o gpurun_out/r2_ritz_gemm python scripts/gemm_bench.py > gpurun_out/ncu_gemm.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_gemm.log
python scripts/cgs2_bench.py "262144,1440" > gpurun_out/cgs2_bench.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rw_stream -c 3 -o gpurun_out/r2_rw_cgs2_k1440 python scripts/cgs2_bench.py "262144,1440" > gpurun_out/ncu_rw.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_rw.log
