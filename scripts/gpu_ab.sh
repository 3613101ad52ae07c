# A/B + profile run on the GPU box (invoked through gpurun)
mkdir -p gpurun_out
rm -f gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 180 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
for pf in 0 1; do
  TG_PREFETCH_ROWS=$pf timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_pf${pf}.log 2>&1; echo "bench pf=$pf rc=$?" >> gpurun_out/status.txt
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 1 -o gpurun_out/prof_fused python bench.py --groups 1 --mb-groups 1 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
