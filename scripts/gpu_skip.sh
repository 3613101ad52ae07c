# phase 1: skip vectors past the slice end for a whole warp (TG_SKIP_EMPTY) -- parity + A/B
mkdir -p gpurun_out/skip
O=gpurun_out/skip
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_tight_parity.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_finite_diff.py > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/status.txt
L=paper_2505_17826_b200/_lib
for rep in 1 2; do
  for v in base noskip; do
    lib=$L/libtg_loss_$v.so; [ $v = base ] && lib=$L/libtg_loss.so
    echo "$v head $(TG_LOSS_LIB=$lib timeout 600 python bench.py --no-e2e --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,3), round(d["roofline"]["frac"],4), d["roofline"]["kernel_ms"], d["clocks"]["sm_mhz"])')" >> $O/ab.txt
    echo "$v anchor $(TG_LOSS_LIB=$lib timeout 300 python scripts/bench_anchor.py | cut -c1-120)" >> $O/ab.txt
  done
done
timeout 900 ncu --set full --clock-control none -k regex:k_fused -c 1 -o $O/grpo python bench.py --groups 2 --mb-groups 1 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu.log 2>&1
TG_LOSS_LIB=$L/libtg_loss_noskip.so timeout 900 ncu --set full --clock-control none -k regex:k_fused -c 1 -o $O/grpo_noskip python bench.py --groups 2 --mb-groups 1 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu2.log 2>&1
