SE_FILTER_CTAS=296 python -m pytest tests/test_gpu_core.py -q -k "apply_pol or spmv" > gpurun_out/t_cap.log 2>&1
for v in "SE_FILTER_CTAS=0" "SE_FILTER_CTAS=296" "SE_FILTER_CTAS=148" "SE_FILTER_CTAS=592" "SE_FILTER_CTAS=296 SE_NO_FILTER_PRIO=1"; do
  echo "== $v" >> gpurun_out/exp3.log
  env $v python scripts/contention_bench.py 2>&1 | head -4 >> gpurun_out/exp3.log
  env $v timeout 300 python scripts/run_cfg.py cfg2 2>&1 | head -1 >> gpurun_out/exp3.log
done
