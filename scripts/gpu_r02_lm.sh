# round-2: native LM-head backward GEMMs (+ one-launch chunk), tight parity, LM-head bench
mkdir -p gpurun_out/lm2
O=gpurun_out/lm2
timeout 900 python -m pytest tests/test_gpu_lmhead.py tests/test_gpu_tight_parity.py -x -q > $O/pytest_lm.txt 2>&1; echo "pytest lm+tight rc=$?" >> $O/status.txt
for dd in 1536 3584; do
  timeout 600 python scripts/bench_lmhead.py --dim $dd >> $O/bench_lmhead.jsonl 2>> $O/bench_lmhead.err; echo "lmhead d=$dd rc=$?" >> $O/status.txt
done
