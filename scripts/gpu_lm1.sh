# LM-head forward A/B (pair / order) at d = 1536 / 3584, ncu of the single-CTA
# forward at d = 3584, sanitizer over the anchor split-stash kernels
mkdir -p gpurun_out/lm1
O=gpurun_out/lm1
L=paper_2505_17826_b200/_lib/libtg_loss_ab.so
for d in 1536 3584; do
  python scripts/ab_lmhead_fwd.py --dim $d --cublas >> $O/ab.jsonl 2>> $O/ab.err
  for pr in 0 1; do for od in 0 1; do
    TG_LOSS_LIB=$L TG_LMHEAD_PAIR=$pr TG_LMHEAD_ORDER=$od timeout 300 python scripts/ab_lmhead_fwd.py --dim $d >> $O/ab.jsonl 2>> $O/ab.err
  done; done
done
timeout 900 ncu --set full --clock-control none -k regex:k_lmhead_logprob -c 1 -o $O/fwd3584 python scripts/ab_lmhead_fwd.py --dim 3584 > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/status.txt
TG_LOSS_LIB=$L TG_LMHEAD_PAIR=1 timeout 900 ncu --set full --clock-control none -k regex:k_lmhead_logprob -c 1 -o $O/fwd3584_pair python scripts/ab_lmhead_fwd.py --dim 3584 > $O/ncu2.log 2>&1; echo "ncu2 rc=$?" >> $O/status.txt
timeout 1200 compute-sanitizer --tool memcheck python scripts/sanitize_small.py anchor > $O/memcheck_anchor.txt 2>&1; echo "memcheck rc=$?" >> $O/status.txt
timeout 1200 compute-sanitizer --tool racecheck python scripts/sanitize_small.py anchor > $O/racecheck_anchor.txt 2>&1; echo "racecheck rc=$?" >> $O/status.txt
timeout 1200 compute-sanitizer --tool synccheck python scripts/sanitize_small.py anchor > $O/synccheck_anchor.txt 2>&1; echo "synccheck rc=$?" >> $O/status.txt
