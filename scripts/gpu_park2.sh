# parked producer / broadcast waits, data waits re-polled (the kept default) vs the previous 64 ns re-polling
mkdir -p gpurun_out/park3
O=gpurun_out/park3
L=paper_2505_17826_b200/_lib
for rep in 1 2 3; do
  for v in base old; do
    lib=$L/libtg_loss_$v.so; [ $v = base ] && lib=$L/libtg_loss.so
    for var in grpo c1; do
      echo "$v $var $(TG_LOSS_LIB=$lib timeout 600 python bench.py --variant $var --no-e2e --no-cpu --steps 8 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,3), round(d["roofline"]["frac"],4), d["clocks"]["sm_mhz"], d["clocks"].get("power_w"))')" >> $O/ab.txt
    done
  done
done
