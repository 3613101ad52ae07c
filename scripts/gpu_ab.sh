# A/B + profile run on the GPU box (invoked through gpurun):
#   bash scripts/gpu_ab.sh [tests] [ncu]   ;  variants via AB_VARIANTS="ENV=1 ENV=2 ..."
mkdir -p gpurun_out
rm -f gpurun_out/status.txt gpurun_out/ab_*.log
if [[ " $* " == *" tests "* ]]; then
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 180 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
fi
i=0
for rep in 1 2; do
  for v in ${AB_VARIANTS:-BASE=1}; do
    i=$((i+1))
    env ${v//,/ } timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ab_${i}_${v}.log 2>&1; echo "bench $v rc=$?" >> gpurun_out/status.txt
  done
done
if [[ " $* " == *" ncu "* ]]; then
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 1 -o gpurun_out/prof_fused python bench.py --groups 1 --mb-groups 1 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
fi
