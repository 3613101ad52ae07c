# round-2 final measurement batch (1 x B200): GPU tests + smoke, headline bench +
# reference arm, every variant, the 2-rank plumbing, launch list, ncu of the
# headline kernel, compute-sanitizer over every kernel
mkdir -p gpurun_out/fin2
O=gpurun_out/fin2
nvidia-smi > $O/nvsmi.txt 2>&1; nproc > $O/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/status.txt
for v in c1 c3 c4 c5 anchor grpo_two_pass opmd_kimi opmd_kimi_unscaled opmd_pairwise_unscaled; do
  timeout 600 python bench.py --variant $v --no-e2e --no-cpu >> $O/variants.jsonl 2>> $O/variants.err; echo "$v rc=$?" >> $O/status.txt
done
TG_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --variant c5 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_gpus2_c5.json 2> $O/bench_gpus2_c5.err; echo "gpus2 c5 rc=$?" >> $O/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $O/launches.log 2>&1; echo "launches rc=$?" >> $O/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 1 -o $O/grpo python bench.py --groups 2 --mb-groups 1 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu_grpo.log 2>&1; echo "ncu grpo rc=$?" >> $O/status.txt
timeout 1500 compute-sanitizer --tool memcheck python scripts/sanitize_small.py > $O/memcheck.txt 2>&1; echo "memcheck rc=$?" >> $O/status.txt
for d in 1536 3584; do timeout 600 python scripts/bench_lmhead.py --dim $d >> $O/lmhead_train.jsonl 2>> $O/lmhead.err; done
for dt in bf16 fp32; do timeout 300 python scripts/bench_adamw.py --dtype $dt >> $O/adamw.jsonl 2>> $O/adamw.err; done
timeout 300 python scripts/bench_anchor.py >> $O/anchor16k.txt 2>&1
