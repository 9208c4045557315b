# A/B of construction compile-time knobs on the GPU box (dev tool): for each
# JB_NVCC_EXTRA variant, rebuild build.cu and time one 100K batch into N rows.
#   bash tools/exp_build_variants.sh N "-DJB_P2_KB=40" ...
set -x
N=$1; shift
for V in "" "$@"; do
  touch paper_2601_07048_b200/csrc/build.cu
  JB_NVCC_EXTRA="$V" python -m paper_2601_07048_b200._build > /dev/null
  JB_PROFILE=1 timeout 600 python tools/prof_donor.py $N 2>&1 | grep "batch \[$N\|batch of" | sed "s/^/VARIANT '$V' /"
done
touch paper_2601_07048_b200/csrc/build.cu
