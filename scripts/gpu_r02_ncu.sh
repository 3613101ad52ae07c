# ncu --set full captures of each variant's dominant kernel (one launch each),
# for profiles/traffic.json and the per-variant profile summaries
mkdir -p gpurun_out/r02ncu
O=gpurun_out/r02ncu
NCU="ncu --set full --clock-control none --import-source on -c 1"
timeout 600 $NCU -k regex:k_fused -o $O/grpo python bench.py --groups 2 --mb-groups 1 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/grpo.log 2>&1; echo "grpo $?" >> $O/status.txt
timeout 600 $NCU -k regex:k_fused -o $O/c1 python bench.py --variant c1 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/c1.log 2>&1; echo "c1 $?" >> $O/status.txt
timeout 600 $NCU -k regex:k_fused -o $O/anchor python bench.py --variant anchor --groups 2 --mb-groups 1 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/anchor.log 2>&1; echo "anchor $?" >> $O/status.txt
