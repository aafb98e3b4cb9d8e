# One `ncu --set full` capture per hot kernel of a 256^3 outer iteration (scripts/profile_step.py),
# reports under gpurun_out/ncu_<tag>_<kernel>.ncu-rep.  usage: bash scripts/ncu_kernels.sh TAG [kernels...]
tag=$1; shift
ks=${@:-"k_fu2d_gather k_fu2d_adj_spread k_fu2d_cols k_fu2d_rows k_fu2d_adj_cols k_fu2d_adj_rows k_fu1d k_fu1d_adj"}
mkdir -p gpurun_out
for k in $ks; do
  memo=off; case $k in k_encode*|k_memo*|k_dev*|k_fu2d_adj_prep) memo=local;; esac
  timeout 300 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"^${k}$" --launch-skip 3 -c 1 -o gpurun_out/ncu_${tag}_${k} -f \
    python scripts/profile_step.py --n ${N:-256} --memo $memo --warmup ${WARMUP:-2} > gpurun_out/ncu_${tag}_${k}.log 2>&1
  echo "$k rc $?"
done
# summaries here (reports with source are too big to bring back all at once)
for k in $ks; do
  r=gpurun_out/ncu_${tag}_${k}.ncu-rep
  [ -f $r ] || continue
  { python scripts/ncu_summary.py $r; echo "# top stalled SASS (scripts/ncu_hot.py)"; python scripts/ncu_hot.py $r 30; } > gpurun_out/ncu_${tag}_${k}.txt 2>&1
  [ -n "$KEEP_REPS" ] || rm -f $r
done
