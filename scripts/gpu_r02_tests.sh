# full GPU test suite + smoke on one B200 (round 2 re-check)
mkdir -p gpurun_out/r02t
O=gpurun_out/r02t
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/status.txt
