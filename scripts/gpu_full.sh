# Full bench (default args, as the driver runs it) + launch list + a full ncu capture of the fused kernel
mkdir -p gpurun_out
rm -f gpurun_out/status_full.txt
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?" >> gpurun_out/status_full.txt
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?" >> gpurun_out/status_full.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/launches.log 2>&1; echo "launches rc=$?" >> gpurun_out/status_full.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status_full.txt
if [[ " $* " == *" ncu "* ]]; then
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 1 -o gpurun_out/prof_fused python bench.py --groups 1 --mb-groups 1 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/status_full.txt
fi
