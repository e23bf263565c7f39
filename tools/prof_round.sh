#!/bin/bash
# One profiling pass (run under gpurun): launch list of the headline bench +
# ncu --set full captures of each hot kernel.  Outputs in gpurun_out/.
O=gpurun_out
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --secondary none > $O/launches_bench.out 2>&1
$NCU --set full --import-source on -k regex:'magnus_fused' -s 1 -c 1 -o $O/magnus2 -f \
    python tools/prof_driver.py magnus2 > $O/magnus2.out 2>&1
$NCU --set full --import-source on -k regex:npad_trows -s 1 -c 1 -o $O/sweep -f \
    python tools/prof_driver.py sweep 1024 > $O/sweep.out 2>&1
$NCU --set full --import-source on -k regex:npad_coop -s 1 -c 1 -o $O/npad4096 -f \
    python tools/prof_driver.py npad4096 2000 > $O/npad4096.out 2>&1
$NCU --set full --import-source on -k regex:'copy_kernel|indptr_kernel' -s 2 -c 2 -o $O/givens -f \
    python tools/prof_driver.py givens 10000000 > $O/givens.out 2>&1
$NCU --set full --import-source on -k regex:npad_full_warp -s 1 -c 1 -o $O/npad60 -f \
    python tools/prof_driver.py npad60 > $O/npad60.out 2>&1
$NCU --set full --import-source on -k regex:zgemm -s 2 -c 2 -o $O/zgemm4096 -f \
    python tools/prof_driver.py magnus4096 > $O/zgemm4096.out 2>&1
$NCU --set full --import-source on -k regex:chain_cta64 -s 1 -c 1 -o $O/midsize -f \
    python tools/midsize_probe.py > $O/midsize.out 2>&1
ls -la $O
