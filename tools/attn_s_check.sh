out=gpurun_out/attns; mkdir -p $out
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_parity_c2.py -q -x > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for n in 1 2 3 6; do timeout 120 python tools/sweep_point.py $n 10 2>&1 | tail -1 | tee -a $out/summary.txt; done
