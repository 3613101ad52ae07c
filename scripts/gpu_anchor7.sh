# anchor KL mode 3: L2 look-ahead by stash positions (TG_PREFETCH_CHUNKS) x copier / geometry
mkdir -p gpurun_out/a7
O=gpurun_out/a7
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_tight_parity.py tests/test_gpu_parity.py -k "anchor" > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/status.txt
L=paper_2505_17826_b200/_lib
for rep in 1 2; do
  for v in ab s4 nocp s4nocp; do
    for pc in 0 4 8 12; do
      echo "$v pc=$pc $(TG_LOSS_LIB=$L/libtg_loss_$v.so TG_PREFETCH_CHUNKS=$pc timeout 300 python scripts/bench_anchor.py)" >> $O/ab.txt
    done
  done
  echo "mode1 $(TG_LOSS_LIB=$L/libtg_loss_ab.so TG_FUSED_ANCHOR_MODE=1 timeout 300 python scripts/bench_anchor.py)" >> $O/ab.txt
done
for pc in 0 8; do
TG_LOSS_LIB=$L/libtg_loss_prof.so TG_PREFETCH_CHUNKS=$pc TG_FUSED_PROF_OUT=$O/prof_m3_$pc.npy timeout 300 python scripts/bench_anchor.py >> $O/prof.txt 2>&1
done
python scripts/prof_report.py 16 $O/prof_m3_0.npy $O/prof_m3_8.npy >> $O/prof.txt 2>&1
