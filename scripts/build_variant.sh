#!/bin/bash
# usage: build_variant.sh NAME "EXTRA_NVFLAGS"  -> paper_2511_01893_b200/libv/NAME/libmlr.so (tuning A/B; MLRG_LIB selects it)
set -e
root=$(cd "$(dirname "$0")/.." && pwd)
make -C "$root/paper_2511_01893_b200/csrc" -j8 BUILD="../build_$1" OUT="../libv/$1" EXTRA_NVFLAGS="$2" >/dev/null
echo "$root/paper_2511_01893_b200/libv/$1/libmlr.so"
