out=gpurun_out/tnck; mkdir -p $out
timeout 1200 python -m pytest tests -q -m gpu -x > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for n in 3 4 6 11 12 16 48; do
  timeout 120 python tools/sweep_point.py $n 10 2>&1 | tail -1 | tee -a $out/summary.txt
done
