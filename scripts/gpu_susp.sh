# suspend-hint waits (power under the cap): base vs consumer data waits parked (suspc) vs every wait parked (susp)
mkdir -p gpurun_out/susp
O=gpurun_out/susp
L=paper_2505_17826_b200/_lib
for rep in 1 2 3; do
  for v in base suspc susp; do
    lib=$L/libtg_loss_$v.so; [ $v = base ] && lib=$L/libtg_loss.so
    echo "$v $(TG_LOSS_LIB=$lib timeout 600 python bench.py --no-e2e --no-cpu --steps 8 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,3), round(d["roofline"]["frac"],4), d["clocks"]["sm_mhz"], d["clocks"].get("power_w"))')" >> $O/ab.txt
  done
done
for v in suspc susp; do echo "$v anchor $(TG_LOSS_LIB=$L/libtg_loss_$v.so timeout 300 python scripts/bench_anchor.py | cut -c1-110)" >> $O/ab.txt; done
echo "base anchor $(timeout 300 python scripts/bench_anchor.py | cut -c1-110)" >> $O/ab.txt
