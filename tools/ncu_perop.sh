#!/bin/bash
# Per-op hardware counters (round 2):
#  (1) PM sampling (time series) of one persistent iteration launch at the bench shape
#  (2) the per-op kernel sequence (ALPA_MK=0): tensor-pipe %, DRAM bytes / throughput per kernel
out=gpurun_out/ncu_perop; mkdir -p $out
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum"
timeout 900 ncu --section PmSampling --section SpeedOfLight --clock-control none -k regex:iter_kernel -s 0 -c 1 \
    -o $out/pm_iter python tools/run_iteration.py --blocks 36 --iters 1 --eager > $out/pm.log 2>&1
ALPA_MK=0 timeout 900 ncu --metrics $M --clock-control none -k regex:'tc_gemm|tc_attn|encode|head|gemm|attn' -s 0 -c 60 --csv \
    --log-file $out/perop.csv python tools/run_iteration.py --blocks 36 --iters 1 --eager > $out/perop.log 2>&1
ALPA_MK=0 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_2605_08975_b200 as alpa
cfg=alpa.ModelConfig(vision_blocks=0,hidden_dim=64,vocab_size=128,decoder_blocks=36,action_hidden_dim=2048,kv_dim=1024,heads=8,diffusion_iters=10,dtype='bf16')
g=alpa.ActionGenerator(cfg); g.bind_prefix_synthetic(4242,2048)
print([ (p['name'],p['launches']) for p in g.profile(alpa.InferenceRequest(num_trajectories=6,v0=5.0),iters=1)])
" > $out/names.txt 2>&1
