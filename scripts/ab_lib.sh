# A/B of prebuilt libraries: bash scripts/ab_lib.sh lib1 lib2 ...  (memo-off 256^3 kernel table each)
for l in "$@"; do
  echo "== $l"
  MLRG_LIB=$PWD/paper_2511_01893_b200/lib/$l timeout 600 python scripts/memo_breakdown.py --n ${N:-256} --steps ${STEPS:-10} --warmup 2 --memo off 2>&1 | grep -E "${PAT:-k_fu2d_adj_spread|kern}" | tail -3
done
