out=gpurun_out/ring; mkdir -p $out
timeout 1200 python -m pytest tests -q -m gpu -x > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for n in 1 6 16; do timeout 120 python tools/sweep_point.py $n 10 2>&1 | tail -1 | tee -a $out/summary.txt; done
ALPA_MK_TRACE=1 timeout 120 python tools/mk_trace.py --blocks 4 > $out/trace6.txt 2>&1
ALPA_MK_TRACE=1 timeout 120 python tools/mk_trace.py --blocks 4 --n 1 > $out/trace1.txt 2>&1
