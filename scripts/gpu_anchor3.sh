# anchor mode 3 (half-size slots) A/B: parity under forced mode 3 / CL 3, then throughput
mkdir -p gpurun_out/an3
O=gpurun_out/an3
L=$PWD/paper_2505_17826_b200/_lib
TG_LOSS_LIB=$L/libtg_loss_ab.so TG_FUSED_ANCHOR_MODE=3 TG_FUSED_CL=3 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "anchor and not fp32" > $O/pytest_m3cl3.txt 2>&1; echo "pytest m3 cl3 rc=$?" >> $O/status.txt
TG_LOSS_LIB=$L/libtg_loss_ab.so TG_FUSED_ANCHOR_MODE=3 TG_FUSED_CL=4 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_anchor_kl_route and v151936" > $O/pytest_m3cl4.txt 2>&1; echo "pytest m3 cl4 rc=$?" >> $O/status.txt
for rep in 1 2; do
  echo "mode1 cl4 $(TG_LOSS_LIB=$L/libtg_loss_ab.so timeout 300 python scripts/bench_anchor.py 151936 16384)" >> $O/ab.txt
  echo "mode3 cl3 $(TG_LOSS_LIB=$L/libtg_loss_ab.so TG_FUSED_ANCHOR_MODE=3 TG_FUSED_CL=3 timeout 300 python scripts/bench_anchor.py 151936 16384)" >> $O/ab.txt
  echo "mode3 cl4 $(TG_LOSS_LIB=$L/libtg_loss_ab.so TG_FUSED_ANCHOR_MODE=3 TG_FUSED_CL=4 timeout 300 python scripts/bench_anchor.py 151936 16384)" >> $O/ab.txt
  echo "mode1 cl3 $(TG_LOSS_LIB=$L/libtg_loss_ab.so TG_FUSED_ANCHOR_MODE=1 TG_FUSED_CL=3 timeout 300 python scripts/bench_anchor.py 151936 16384)" >> $O/ab.txt
  echo "V=65536 mode1 cl2 $(TG_LOSS_LIB=$L/libtg_loss_ab.so timeout 300 python scripts/bench_anchor.py 65536 32768)" >> $O/ab.txt
  echo "V=65536 mode3 cl2 $(TG_LOSS_LIB=$L/libtg_loss_ab.so TG_FUSED_ANCHOR_MODE=3 TG_FUSED_CL=2 timeout 300 python scripts/bench_anchor.py 65536 32768)" >> $O/ab.txt
done
