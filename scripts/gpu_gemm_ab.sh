# backward GEMMs: pair vs single CTAs, interleaved, 3 repetitions, d = 1536 / 3584
mkdir -p gpurun_out/gab
O=gpurun_out/gab
L=paper_2505_17826_b200/_lib/libtg_loss_ab.so
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv >> $O/clocks.txt
for rep in 1 2 3; do
  for d in 1536 3584; do
    for m in 1 0; do
      TG_LOSS_LIB=$L TG_GEMM_PAIR=$m timeout 300 python scripts/ab_gemm.py --dim $d >> $O/ab.jsonl 2>> $O/ab.err
    done
  done
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv >> $O/clocks.txt
