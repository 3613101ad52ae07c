# backward GEMMs as 2-CTA pairs: parity (both CTA modes), training-step bench
mkdir -p gpurun_out/lm4
O=gpurun_out/lm4
timeout 1200 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_lmhead.py > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/status.txt
for d in 1536 3584; do timeout 600 python scripts/bench_lmhead.py --dim $d >> $O/lmhead_train.jsonl 2>> $O/lmhead.err; done
for d in 1536 3584; do TG_LOSS_LIB=paper_2505_17826_b200/_lib/libtg_loss_ab.so TG_GEMM_PAIR=0 timeout 600 python scripts/bench_lmhead.py --dim $d >> $O/lmhead_train_single.jsonl 2>> $O/lmhead.err; done
timeout 900 ncu --set full --clock-control none -k regex:k_gemm -c 1 -o $O/gemm_pair python scripts/bench_lmhead.py --rows 16384 > $O/ncu_gemm.log 2>&1; echo "ncu rc=$?" >> $O/status.txt
