# backward GEMM pairs: 6 vs 7 shared-memory stages, interleaved, 3 repetitions
mkdir -p gpurun_out/gab2
O=gpurun_out/gab2
for rep in 1 2 3; do
  for d in 1536 3584; do
    for v in ab g7; do
      TG_LOSS_LIB=paper_2505_17826_b200/_lib/libtg_loss_$v.so timeout 300 python scripts/ab_gemm.py --dim $d | sed "s/^/$v /" >> $O/ab.txt 2>> $O/ab.err
    done
  done
done
