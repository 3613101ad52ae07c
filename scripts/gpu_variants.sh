# full GPU tests + bench of the headline and the two-pass / coupled routes
mkdir -p gpurun_out
rm -f gpurun_out/status_var.txt gpurun_out/var_*.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status_var.txt
for v in ${VARIANTS:-grpo grpo_two_pass opmd_kimi}; do
  timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --variant $v > gpurun_out/var_$v.log 2>&1; echo "bench $v rc=$?" >> gpurun_out/status_var.txt
done
