# A/B of prebuilt library variants (paper_2505_17826_b200/_lib/libtg_loss_<name>.so;
# "base" = libtg_loss.so) on the headline bench.
#   LIBS="base p1 base:TG_FUSED_CL=3,TG_X=1" REPS=2 STEPS=3 BENCH_ARGS="..."
mkdir -p gpurun_out
rm -f gpurun_out/libab_*.json gpurun_out/libab_*.err gpurun_out/libab_status.txt
for rep in $(seq 1 ${REPS:-2}); do
  for spec in ${LIBS:-base}; do
    v=${spec%%:*}
    envs=""; [ "$spec" != "$v" ] && envs=${spec#*:}
    tag=$(echo "$spec" | tr ':,=' '___')
    lib=$PWD/paper_2505_17826_b200/_lib/libtg_loss_$v.so
    [ "$v" = base ] && lib=$PWD/paper_2505_17826_b200/_lib/libtg_loss.so
    env ${envs//,/ } TG_LOSS_LIB=$lib timeout 300 python bench.py --steps ${STEPS:-3} --warmup 2 \
      --no-cpu --no-e2e ${BENCH_ARGS:-} > gpurun_out/libab_${tag}_$rep.json 2> gpurun_out/libab_${tag}_$rep.err
    echo "$spec rep$rep rc=$?" >> gpurun_out/libab_status.txt
  done
done
python scripts/libab_report.py gpurun_out/libab_*.json
