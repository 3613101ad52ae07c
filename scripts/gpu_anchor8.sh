# anchor KL mode 3 default (consumer copy + L2 look-ahead by positions): parity,
# cycle accounting, ncu, bench line
mkdir -p gpurun_out/a8
O=gpurun_out/a8
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_tight_parity.py tests/test_gpu_parity.py tests/test_gpu_alt_paths.py tests/test_gpu_fuzz.py -k "anchor or fuzz" > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/status.txt
L=paper_2505_17826_b200/_lib
for pc in 0 2 4 6 8; do
  echo "base pc=$pc $(TG_LOSS_LIB=$L/libtg_loss_ab.so TG_PREFETCH_CHUNKS=$pc timeout 300 python scripts/bench_anchor.py)" >> $O/ab.txt
done
echo "default $(timeout 300 python scripts/bench_anchor.py)" >> $O/ab.txt
echo "mode1 $(TG_LOSS_LIB=$L/libtg_loss_ab.so TG_FUSED_ANCHOR_MODE=1 timeout 300 python scripts/bench_anchor.py)" >> $O/ab.txt
for pc in 0 6; do
TG_LOSS_LIB=$L/libtg_loss_prof.so TG_PREFETCH_CHUNKS=$pc TG_FUSED_PROF_OUT=$O/prof_m3_$pc.npy timeout 300 python scripts/bench_anchor.py >> $O/prof.txt 2>&1
done
python scripts/prof_report.py 16 $O/prof_m3_0.npy $O/prof_m3_6.npy >> $O/prof.txt 2>&1
timeout 600 python bench.py --variant anchor --no-e2e --no-cpu > $O/bench_anchor.json 2> $O/bench_anchor.err; echo "bench rc=$?" >> $O/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 1 -o $O/anchor python scripts/bench_anchor.py > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/status.txt
