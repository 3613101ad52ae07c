# backward GEMMs: tail split (last partial wave as half tiles) on / off; parity in both CTA modes
mkdir -p gpurun_out/gt
O=gpurun_out/gt
timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_lmhead.py > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/status.txt
L=paper_2505_17826_b200/_lib/libtg_loss_ab.so
for rep in 1 2 3; do
  for d in 1536 3584; do
    for t in 1 0; do
      TG_LOSS_LIB=$L TG_GEMM_TAIL=$t timeout 300 python scripts/ab_gemm.py --dim $d | sed "s/^/tail=$t /" >> $O/ab.txt 2>> $O/ab.err
    done
  done
done
