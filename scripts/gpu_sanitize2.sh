# compute-sanitizer over the LM-head paths (2-CTA forward, dz chunks, pair GEMMs) and the fused AdamW
mkdir -p gpurun_out/san2
O=gpurun_out/san2
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool python scripts/sanitize_small.py lmhead > $O/${tool}_lmhead.txt 2>&1; echo "$tool lmhead rc=$?" >> $O/status.txt
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_small.py optim > $O/${tool}_optim.txt 2>&1; echo "$tool optim rc=$?" >> $O/status.txt
done
timeout 1500 compute-sanitizer --tool initcheck python scripts/sanitize_small.py optim > $O/initcheck_optim.txt 2>&1; echo "initcheck optim rc=$?" >> $O/status.txt
