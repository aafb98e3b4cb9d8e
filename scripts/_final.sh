python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?
P="ncu --profile-from-start off --clock-control none"
timeout 600 $P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r1_launches_step256.csv python scripts/profile_step.py --n 256 > /dev/null 2>&1
timeout 600 $P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r1_launches_step256_memo.csv python scripts/profile_step.py --n 256 --memo local --warmup 3 > /dev/null 2>&1
timeout 600 $P --set full --import-source on -k regex:k_fu2d_gather -c 1 -o gpurun_out/r1_k_fu2d_gather python scripts/profile_step.py --n 256 > /dev/null 2>&1
ls gpurun_out/r1_k_fu2d_gather.ncu-rep
