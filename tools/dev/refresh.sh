# end-of-round refresh: GPU tests, smoke, bench lines, launch lists (run under gpurun)
set -x
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k "regex:tf_" --csv python tools/time_fold.py > $O/launches_fold.csv 2> $O/launches_fold.err
timeout 420 python tools/fuzz.py 360 43 > $O/fuzz_seed43.log 2>&1
