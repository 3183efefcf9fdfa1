#!/bin/bash
# Variant builds for the per-choice ncu before/after table (tools/ncu_choices.sh): each turns ONE choice off.
set -e
cd "$(dirname "$0")/.."
bash tools/build_variant.sh no_black "-DFHT_P2_BLACK=0"
bash tools/build_variant.sh no_scr_keep "-DFHT_SCR_KEEP=0"
bash tools/build_variant.sh no_warpload "-DFHT_P2_WARPLOAD=0 -DFHT_P1_WARPLOAD=0"
bash tools/build_variant.sh no_dense "-DFHT_P2_DENSE=0"
bash tools/build_variant.sh no_unpred "-DFHT_P2_UNPRED=0"
bash tools/build_variant.sh no_stage2 "-DFHT_P1_STAGE2=0"
bash tools/build_variant.sh no_dense_mask "-DFHT_P2_DENSE_MASK=0"
bash tools/build_variant.sh no_pdl "-DFHT_PDL=0"
ls -la build/ab
