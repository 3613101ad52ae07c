# anchor KL mode 3 geometry A/B: shared stash slots 5 / 4 / 3 (landing 2 / 3 / 4),
# L2 row prefetch, and the instrumented cycle accounting of modes 1 and 3
mkdir -p gpurun_out/a5
O=gpurun_out/a5
L=paper_2505_17826_b200/_lib
for rep in 1 2; do
  for v in ab s4 s3; do
    for pf in 0 1; do
      echo "$v pf=$pf $(TG_LOSS_LIB=$L/libtg_loss_$v.so TG_PREFETCH_ROWS=$pf timeout 300 python scripts/bench_anchor.py)" >> $O/ab.txt
    done
  done
  echo "mode1 $(TG_LOSS_LIB=$L/libtg_loss_ab.so TG_FUSED_ANCHOR_MODE=1 timeout 300 python scripts/bench_anchor.py)" >> $O/ab.txt
done
TG_LOSS_LIB=$L/libtg_loss_prof.so TG_FUSED_PROF_OUT=$O/prof_m3.npy timeout 300 python scripts/bench_anchor.py >> $O/prof.txt 2>&1
TG_LOSS_LIB=$L/libtg_loss_prof.so TG_FUSED_ANCHOR_MODE=1 TG_FUSED_PROF_OUT=$O/prof_m1.npy timeout 300 python scripts/bench_anchor.py >> $O/prof.txt 2>&1
python scripts/prof_report.py 16 $O/prof_m3.npy $O/prof_m1.npy >> $O/prof.txt 2>&1
