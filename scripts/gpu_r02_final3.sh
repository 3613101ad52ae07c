# final tree (after the phase-1 empty-vector skip): 1,000-seed fuzz, headline bench + variants
mkdir -p gpurun_out/fin3b
O=gpurun_out/fin3b
TG_FUZZ_SEEDS=1000 timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_gpu_fuzz.py > $O/fuzz.txt 2>&1; echo "fuzz rc=$?" >> $O/status.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
for v in c1 c3 c4 c5 anchor grpo_two_pass opmd_kimi_unscaled; do
  timeout 600 python bench.py --variant $v --no-e2e --no-cpu >> $O/variants.jsonl 2>> $O/variants.err; echo "$v rc=$?" >> $O/status.txt
done
