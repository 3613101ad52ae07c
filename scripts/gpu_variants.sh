# bench the non-headline routes (two-pass / sequence-coupled) + packer tests
mkdir -p gpurun_out
rm -f gpurun_out/status_var.txt gpurun_out/var_*.log
timeout 600 python -m pytest tests/test_gpu_packer.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "packer or config" > gpurun_out/pytest_var.log 2>&1; echo pytest=$? >> gpurun_out/status_var.txt
for v in ${VARIANTS:-grpo grpo_two_pass opmd_kimi}; do
  timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --variant $v > gpurun_out/var_$v.log 2>&1; echo "bench $v rc=$?" >> gpurun_out/status_var.txt
done
