# LM-head tcgen05 kernels: parked waits (TG_LM_PARK) vs spin / 32 ns re-poll; forward + GEMM timings
mkdir -p gpurun_out/lmpark
O=gpurun_out/lmpark
L=paper_2505_17826_b200/_lib
for rep in 1 2 3; do
  for v in base lmpark; do
    lib=$L/libtg_loss_$v.so; [ $v = base ] && lib=$L/libtg_loss.so
    for d in 1536 3584; do
      echo "$v fwd $(TG_LOSS_LIB=$lib timeout 300 python scripts/ab_lmhead_fwd.py --dim $d)" >> $O/ab.txt
      echo "$v gemm $(TG_LOSS_LIB=$lib timeout 300 python scripts/ab_gemm.py --dim $d)" >> $O/ab.txt
    done
  done
done
TG_LOSS_LIB=$L/libtg_loss_lmpark.so timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_lmhead.py > $O/pytest.txt 2>&1; echo rc=$? >> $O/pytest.txt
