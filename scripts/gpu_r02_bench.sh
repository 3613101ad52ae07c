# round-2 measurement batch: headline bench, configs, multi-rank plumbing,
# reference arm, c1 timeline
mkdir -p gpurun_out/r02
O=gpurun_out/r02
nvidia-smi > $O/nvsmi.txt 2>&1; nproc > $O/nproc.txt; free -g >> $O/nproc.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
for v in ${VARIANTS:-c1 c3 c5}; do
  timeout 600 python bench.py --variant $v --no-e2e > $O/bench_$v.json 2> $O/bench_$v.err; echo "$v rc=$?" >> $O/status.txt
done
timeout 600 python bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu > $O/bench_gpus2.json 2> $O/bench_gpus2.err; echo "gpus2 rc=$?" >> $O/status.txt
timeout 600 python bench.py --gpus 2 --variant c3 --steps 2 --warmup 1 --no-cpu > $O/bench_gpus2_c3.json 2> $O/bench_gpus2_c3.err; echo "gpus2 c3 rc=$?" >> $O/status.txt
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/status.txt
timeout 300 python scripts/prof_timeline.py > $O/c1_timeline.txt 2>&1; echo "timeline rc=$?" >> $O/status.txt
