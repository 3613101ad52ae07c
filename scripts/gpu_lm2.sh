# LM head with 2-CTA pairs by default (forward too): parity, the training-step
# bench at d = 1536 / 3584; racecheck of the anchor split stash with every
# thread arriving (sanitizer classification)
mkdir -p gpurun_out/lm2
O=gpurun_out/lm2
timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_lmhead.py tests/test_gpu_alt_paths.py > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/status.txt
for d in 1536 3584; do timeout 600 python scripts/bench_lmhead.py --dim $d >> $O/lmhead_train.jsonl 2>> $O/lmhead.err; done
TG_LOSS_LIB=paper_2505_17826_b200/_lib/libtg_loss_arriveall.so timeout 1200 compute-sanitizer --tool racecheck python scripts/sanitize_small.py anchor > $O/racecheck_anchor_arriveall.txt 2>&1; echo "racecheck rc=$?" >> $O/status.txt
