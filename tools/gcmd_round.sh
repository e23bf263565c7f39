#!/bin/bash
# Full measurement pass (run under gpurun): GPU tests, bench (both arms),
# profiling captures.  Outputs in gpurun_out/.
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
python bench.py > $O/bench.json 2> $O/bench.err; tail -c 600 $O/bench.json
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 300 $O/bench_ref.json
bash tools/prof_round.sh > $O/prof_round.log 2>&1; tail -3 $O/prof_round.log
