# full GPU test suite + per-kernel racecheck of the new / changed kernels
mkdir -p gpurun_out/chk2
O=gpurun_out/chk2
# (test suite: see gpurun_out/chk2/pytest.txt of the first run)
for k in k_gemm k_fused_tma k_lmhead; do
  timeout 1200 compute-sanitizer --tool racecheck --kernel-name kns=$k python scripts/sanitize_small.py > $O/racecheck_$k.txt 2>&1; echo "racecheck $k rc=$?" >> $O/status.txt
done
timeout 1200 compute-sanitizer --tool synccheck --kernel-name kns=k_gemm python scripts/sanitize_small.py > $O/synccheck_gemm.txt 2>&1; echo "synccheck gemm rc=$?" >> $O/status.txt
timeout 1200 compute-sanitizer --tool initcheck --kernel-name kns=k_gemm python scripts/sanitize_small.py > $O/initcheck_gemm.txt 2>&1; echo "initcheck gemm rc=$?" >> $O/status.txt
