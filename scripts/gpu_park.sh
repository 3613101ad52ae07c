# parked waits (new defaults) vs the previous 64 ns re-polling: headline, c1, two-pass, anchor + parity
mkdir -p gpurun_out/park
O=gpurun_out/park
timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_tight_parity.py tests/test_gpu_parity.py tests/test_gpu_properties.py > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/status.txt
L=paper_2505_17826_b200/_lib
for rep in 1 2 3; do
  for v in base old; do
    lib=$L/libtg_loss_$v.so; [ $v = base ] && lib=$L/libtg_loss.so
    for var in grpo c1 grpo_two_pass; do
      echo "$v $var $(TG_LOSS_LIB=$lib timeout 600 python bench.py --variant $var --no-e2e --no-cpu --steps 8 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,3), round(d["roofline"]["frac"],4), d["clocks"]["sm_mhz"], d["clocks"].get("power_w"))')" >> $O/ab.txt
    done
    echo "$v anchor $(TG_LOSS_LIB=$lib timeout 300 python scripts/bench_anchor.py | cut -c40-110)" >> $O/ab.txt
  done
done
