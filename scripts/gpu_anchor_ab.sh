# A/B of the fused anchor path and the epilogue merge (scripts/bench_anchor.py),
# plus instrumented per-row cycle accounting of both merge forms.  Build the
# variants first:
#   python -m paper_2505_17826_b200._build --variant=mergeold --define=-DTG_MERGE_REDUX=0
#   python -m paper_2505_17826_b200._build --variant=prof
#   python -m paper_2505_17826_b200._build --variant=profold --define=-DTG_FUSED_PROF --define=-DTG_MERGE_REDUX=0
mkdir -p gpurun_out
L=$PWD/paper_2505_17826_b200/_lib
for rep in 1 2; do
  for v in "" _mergeold; do
    for V in 151936 32000; do
      R=16384; [ $V = 32000 ] && R=65536
      echo "lib=base$v V=$V $(TG_LOSS_LIB=$L/libtg_loss$v.so timeout 300 python scripts/bench_anchor.py $V $R)"
    done
  done
done
for v in prof profold; do
  TG_LOSS_LIB=$L/libtg_loss_$v.so TG_FUSED_PROF_OUT=gpurun_out/pa_$v.npy timeout 300 python scripts/bench_anchor.py > /dev/null
  TG_LOSS_LIB=$L/libtg_loss_$v.so TG_FUSED_PROF_OUT=gpurun_out/pg_$v.npy timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
done
python scripts/prof_report.py 16 gpurun_out/pa_prof.npy gpurun_out/pa_profold.npy gpurun_out/pg_prof.npy gpurun_out/pg_profold.npy
