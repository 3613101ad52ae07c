# phase-2 clamp only in rows whose phase 1 took the checked path: parity + A/B
mkdir -p gpurun_out/clamp
O=gpurun_out/clamp
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_tight_parity.py tests/test_gpu_fuzz.py tests/test_gpu_finite_diff.py > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/status.txt
L=paper_2505_17826_b200/_lib
for rep in 1 2; do
  echo "new anchor $(timeout 300 python scripts/bench_anchor.py)" >> $O/ab.txt
  echo "old anchor $(TG_LOSS_LIB=$L/libtg_loss_clampall.so timeout 300 python scripts/bench_anchor.py)" >> $O/ab.txt
  echo "new c3 $(timeout 600 python bench.py --variant c3 --no-e2e --no-cpu --steps 3 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"])')" >> $O/ab.txt
  echo "old c3 $(TG_LOSS_LIB=$L/libtg_loss_clampall.so timeout 600 python bench.py --variant c3 --no-e2e --no-cpu --steps 3 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"])')" >> $O/ab.txt
done
