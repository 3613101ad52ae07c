# anchor mode 2 (z stashed, za re-read from L2): parity, A/B vs mode 1, ncu, bench
mkdir -p gpurun_out/an2
O=gpurun_out/an2
L=$PWD/paper_2505_17826_b200/_lib
timeout 900 python -m pytest tests/test_gpu_tight_parity.py tests/test_gpu_parity.py -x -q -k "anchor or headline" > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/status.txt
for rep in 1 2; do
  for m in 1 2; do
    echo "mode=$m $(TG_LOSS_LIB=$L/libtg_loss_ab.so TG_FUSED_ANCHOR_MODE=$m timeout 300 python scripts/bench_anchor.py 151936 16384)" >> $O/ab.txt
  done
  echo "mode=2 za_evict_normal $(TG_LOSS_LIB=$L/libtg_loss_zanorm.so timeout 300 python scripts/bench_anchor.py 151936 16384)" >> $O/ab.txt
  for m in 1 2; do
    echo "V=65536 mode=$m $(TG_LOSS_LIB=$L/libtg_loss_ab.so TG_FUSED_ANCHOR_MODE=$m timeout 300 python scripts/bench_anchor.py 65536 32768)" >> $O/ab.txt
  done
done
timeout 600 python bench.py --variant anchor --no-e2e > $O/bench_anchor.json 2> $O/bench_anchor.err; echo "bench anchor rc=$?" >> $O/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -c 1 -k regex:k_fused -o $O/anchor python bench.py --variant anchor --groups 2 --mb-groups 1 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/status.txt
timeout 600 python bench.py --no-cpu > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
