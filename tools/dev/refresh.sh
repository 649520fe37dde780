# end-of-round refresh: GPU tests, bench lines, launch lists (run under gpurun)
set -x
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
for C in C3 C4 C2; do python bench.py --config $C > $O/bench_$C.json 2> $O/bench_$C.err; done
for C in C5 C3 C4; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k "regex:fz_|sh_|sc_" --csv python bench.py --config $C --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-calls \
      > $O/launches_$C.csv 2> $O/launches_$C.err
done
timeout 420 python tools/fuzz.py 360 41 > $O/fuzz_seed41.log 2>&1
