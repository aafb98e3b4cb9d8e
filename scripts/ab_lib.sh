# A/B of prebuilt libraries: bash scripts/ab_lib.sh lib1 lib2 ...  (memo-off 256^3 kernel table each)
for l in "$@"; do
  echo "== $l"
  MLRG_LIB=$PWD/paper_2511_01893_b200/lib/$l timeout 600 python scripts/memo_breakdown.py --steps 10 --memo off 2>&1 | grep -E "k_fu2d_adj_spread|kern" | tail -3
done
