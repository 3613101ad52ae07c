# anchor KL mode 3 (split stash, 2-CTA clusters on 148 SMs): parity + A/B against modes 1 / 2
mkdir -p gpurun_out/a4
O=gpurun_out/a4
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_tight_parity.py tests/test_gpu_alt_paths.py "tests/test_gpu_parity.py" -k "anchor" > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/status.txt
AB=paper_2505_17826_b200/_lib/libtg_loss_ab.so
for rep in 1 2; do
  echo "mode3 $(timeout 300 python scripts/bench_anchor.py)" >> $O/ab.txt
  echo "mode1 $(TG_LOSS_LIB=$AB TG_FUSED_ANCHOR_MODE=1 timeout 300 python scripts/bench_anchor.py)" >> $O/ab.txt
  echo "mode2 $(TG_LOSS_LIB=$AB TG_FUSED_ANCHOR_MODE=2 timeout 300 python scripts/bench_anchor.py)" >> $O/ab.txt
done
timeout 600 python bench.py --variant anchor --no-e2e --no-cpu > $O/bench_anchor.json 2> $O/bench_anchor.err; echo "bench rc=$?" >> $O/status.txt
