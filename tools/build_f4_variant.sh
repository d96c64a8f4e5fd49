#!/bin/bash
# Variant of the library with ALL single-pass sweep translation units (k_fused4*.cu) rebuilt
# with extra nvcc flags:   tools/build_f4_variant.sh <name> <nvcc flags...>   -> build_ab/<name>.so
#   e.g. tools/build_f4_variant.sh f4check -DBIC_F4_CHECK     (protocol-check build)
#        tools/build_f4_variant.sh f4trace -DBIC_F4_TRACE     (per-batch clock64 timeline)
set -e
NAME=$1; shift
cd "$(dirname "$0")/.."
python -c "import paper_2405_16267_b200.build as b; b.build()" > /dev/null
mkdir -p build_ab
ARCH="-gencode arch=compute_100a,code=sm_100a"
INC=$(python -c "import paper_2405_16267_b200.build as b; print(' '.join(b._nccl_include()))")
OBJS=""
for f in paper_2405_16267_b200/csrc/k_fused4*.cu; do
  o=build_ab/${NAME}_$(basename ${f%.cu}).o
  nvcc $ARCH -O3 -lineinfo -std=c++17 --extended-lambda -Xcompiler -fPIC -Iinclude $INC "$@" -c $f -o $o &
  OBJS="$OBJS $o"
done
wait
KEEP=$(ls paper_2405_16267_b200/build/*.o | grep -v "/k_fused4")
nvcc $ARCH -shared -o build_ab/$NAME.so $KEEP $OBJS -ldl
echo build_ab/$NAME.so
