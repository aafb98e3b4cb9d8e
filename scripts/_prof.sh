P="ncu --profile-from-start off --clock-control none"
timeout 600 $P --set full --import-source on -k regex:k_fu2d_gather -c 1 -o gpurun_out/r1_k_fu2d_gather python scripts/profile_step.py --n 256 > /dev/null 2>&1
timeout 600 $P --set full --import-source on -k regex:k_encode -c 1 -o gpurun_out/r1_k_encode python scripts/profile_step.py --n 256 --memo local --warmup 3 > /dev/null 2>&1
timeout 600 $P --set full --import-source on -k regex:k_memo_lookup -c 1 -o gpurun_out/r1_k_memo_lookup python scripts/profile_step.py --n 256 --memo local --warmup 8 > /dev/null 2>&1
timeout 600 $P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r1_launches_step256.csv python scripts/profile_step.py --n 256 > /dev/null 2>&1
timeout 600 $P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r1_launches_step256_memo.csv python scripts/profile_step.py --n 256 --memo local --warmup 3 > /dev/null 2>&1
ls -la gpurun_out/r1_k_* gpurun_out/r1_launches*
