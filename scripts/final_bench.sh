# Round-end measurement set: default bench line, launch list of one 256^3 iteration (memo off / on),
# per-kernel ncu summaries. Writes gpurun_out/.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_off.csv python scripts/profile_step.py --n 256 --memo off > /dev/null 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_memo.csv python scripts/profile_step.py --n 256 --memo local --warmup 5 > /dev/null 2>&1
python scripts/launch_agg.py gpurun_out/launches_off.csv > gpurun_out/launch_summary_off.txt 2>&1
python scripts/launch_agg.py gpurun_out/launches_memo.csv > gpurun_out/launch_summary_memo.txt 2>&1
timeout 300 python scripts/timeline.py --memo off --warmup 4 --steps 2 --out gpurun_out/timeline_off.txt > gpurun_out/timeline_off_summary.txt 2>&1
timeout 300 python scripts/timeline.py --memo local --warmup 4 --steps 2 --out gpurun_out/timeline_memo.txt > gpurun_out/timeline_memo_summary.txt 2>&1
bash scripts/ncu_kernels.sh final k_fu2d_gather k_fu2d_adj_spread k_fu2d_cols k_fu2d_rows k_fu2d_adj_cols k_fu2d_adj_rows k_fu1d k_fu1d_adj k_encode_tc
python -c "import json; d=json.load(open('gpurun_out/bench_final.json')); print(d['value'], d['memo_on']['value'], d['e2e']['value'])"
