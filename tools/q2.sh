# dev loop: trace (with dump) + bench.  bash tools/q2.sh tag
tag=$1; out=gpurun_out/$tag; mkdir -p $out
ALPA_MK_TRACE=1 timeout 120 python tools/mk_trace.py --blocks 4 --extra --dump $out/tr.npz > $out/tr.txt 2>&1
timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/b.json 2> $out/b.err
python -c "import json;d=json.load(open('$out/b.json'));print('ms/scene', d['ms_per_step'])" | tee $out/ms.txt
