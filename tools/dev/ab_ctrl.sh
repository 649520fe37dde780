python tools/dev/fz_quick.py check > gpurun_out/c.log 2>&1
python -m pytest tests/test_gpu_fused.py tests/test_gpu_fused_shard.py tests/test_gpu_scene.py -x -q > gpurun_out/pt.log 2>&1
python tools/dev/fz_quick.py time > gpurun_out/t1.log 2>&1
python tools/dev/fz_quick.py time 24 > gpurun_out/t24.log 2>&1
for C in C3 C4 C5; do echo "$C $(python bench.py --config $C --no-cpu-baseline --no-e2e --no-calls --steps 10 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["roofline"]["per_kernel_ms"])')" >> gpurun_out/ab.txt; done
