# anchor KL mode 3 with the tcgen05.cp copier: parity, then geometry A/B
mkdir -p gpurun_out/a6
O=gpurun_out/a6
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_tight_parity.py tests/test_gpu_parity.py -k "anchor" > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/status.txt
L=paper_2505_17826_b200/_lib
for rep in 1 2; do
  for v in ab s4 s6 s4nocp; do
    for pf in 0 1; do
      echo "$v pf=$pf $(TG_LOSS_LIB=$L/libtg_loss_$v.so TG_PREFETCH_ROWS=$pf timeout 300 python scripts/bench_anchor.py)" >> $O/ab.txt
    done
  done
  echo "mode1 $(TG_LOSS_LIB=$L/libtg_loss_ab.so TG_FUSED_ANCHOR_MODE=1 timeout 300 python scripts/bench_anchor.py)" >> $O/ab.txt
done
TG_LOSS_LIB=$L/libtg_loss_prof.so TG_FUSED_PROF_OUT=$O/prof_m3.npy timeout 300 python scripts/bench_anchor.py >> $O/prof.txt 2>&1
python scripts/prof_report.py 16 $O/prof_m3.npy >> $O/prof.txt 2>&1
