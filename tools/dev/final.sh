# final verification of the committed code (run under gpurun)
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k "regex:fz_|sh_|sc_" --csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-calls \
    > $O/launches_C5.csv 2> $O/launches_C5.err
timeout 480 python tools/fuzz.py 360 67 > $O/fuzz_seed67.log 2>&1
for C in C3 C4 C2; do python bench.py --config $C > $O/bench_$C.json 2> $O/bench_$C.err; done
