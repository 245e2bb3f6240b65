set -x
mkdir -p gpurun_out/p1
./tools/gemm_bench > gpurun_out/p1/gemm_bench.txt 2>&1
# full capture: mlp1 none (launch 4 of first config), mlp1 ln_gelu, mlp2 resid S=4
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 10 -c 1 -o gpurun_out/p1/mlp1_none ./tools/gemm_bench > gpurun_out/p1/ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 220 -c 1 -o gpurun_out/p1/mlp1_lngelu ./tools/gemm_bench > gpurun_out/p1/ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn_kernel -s 20 -c 1 -o gpurun_out/p1/attn python tools/run_iteration.py --blocks 2 --iters 10 --eager > gpurun_out/p1/ncu3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 40 -c 4 -o gpurun_out/p1/blockgemms python tools/run_iteration.py --blocks 2 --iters 10 --eager > gpurun_out/p1/ncu4.log 2>&1
echo done
