#!/bin/bash
# A/B variant of the library with the single-pass sweep sources (k_fused4*) of another commit:
#   tools/build_commit_variant.sh <commit> <name>   -> build_ab/<name>.so  (BICADMM_LIB_PATH selects it)
set -e
C=$1; NAME=$2
cd "$(dirname "$0")/.."
python -c "import paper_2405_16267_b200.build as b; b.build()" > /dev/null
T=$(mktemp -d)
mkdir -p $T/csrc build_ab
git archive $C paper_2405_16267_b200/csrc include | tar -x -C $T
ARCH="-gencode arch=compute_100a,code=sm_100a"
INC=$(python -c "import paper_2405_16267_b200.build as b; print(' '.join(b._nccl_include()))")
OBJS=""
for f in $T/paper_2405_16267_b200/csrc/k_fused4*.cu; do
  o=$T/$(basename ${f%.cu}).o
  nvcc $ARCH -O3 -lineinfo -std=c++17 --extended-lambda -Xcompiler -fPIC -I$T/include $INC -c $f -o $o &
  OBJS="$OBJS $o"
done
wait
KEEP=$(ls paper_2405_16267_b200/build/*.o | grep -v "/k_fused4")
nvcc $ARCH -shared -o build_ab/$NAME.so $KEEP $OBJS -ldl
rm -rf $T
echo build_ab/$NAME.so
