#!/bin/bash
# Final profiling pass of round 2 (run under gpurun, one GPU): launch list of
# the bench + ncu --set full captures of each hot kernel -> gpurun_out/,
# summarised on the box (reports are large).
O=gpurun_out
mkdir -p $O
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --secondary none > $O/launches_bench.out 2>&1
$NCU --set full --import-source on -k regex:'magnus_fused' -s 1 -c 1 -o $O/magnus2 -f \
    python tools/prof_driver.py magnus2 > $O/magnus2.out 2>&1
$NCU --set full --import-source on -k regex:'oz_' -s 6 -c 6 -o $O/oz -f \
    python tools/oz_herm_probe.py 1 > $O/oz.out 2>&1
$NCU --set full --import-source on -k regex:'zgemm_tma' -s 1 -c 1 -o $O/zgemm4096 -f \
    python tools/prof_driver.py zgemm4096 > $O/zgemm4096.out 2>&1
$NCU --set full --import-source on -k regex:npad_trows_warp -s 1 -c 1 -o $O/sweep -f \
    python tools/prof_driver.py sweep 1024 > $O/sweep.out 2>&1
$NCU --set full --import-source on -k regex:npad_coop -s 1 -c 1 -o $O/npad4096 -f \
    python tools/prof_driver.py npad4096 2000 > $O/npad4096.out 2>&1
python tools/ncu_summary.py $O/ncu_full_final.md $O/magnus2.ncu-rep $O/oz.ncu-rep $O/zgemm4096.ncu-rep \
    $O/sweep.ncu-rep $O/npad4096.ncu-rep > $O/summary.log 2>&1
python tools/ncu_summary.py --launches $O/launches_bench_final.md $O/launches_bench.csv >> $O/summary.log 2>&1
cp profiles/ncu_traffic.json $O/ncu_traffic.json
find $O -name '*.ncu-rep' -delete
ls -la $O
