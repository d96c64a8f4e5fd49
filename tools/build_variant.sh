#!/bin/bash
# A/B variant of the library: recompile one source with extra nvcc flags and link it with the
# package's current objects into build_ab/<name>.so (BICADMM_LIB_PATH selects it).
#   tools/build_variant.sh <name> <source.cu> <nvcc flags...>
set -e
NAME=$1; SRC=$2; shift 2
cd "$(dirname "$0")/.."
python -c "import paper_2405_16267_b200.build as b; b.build()" > /dev/null
OBJ=paper_2405_16267_b200/build
mkdir -p build_ab
ARCH="-gencode arch=compute_100a,code=sm_100a"
INC=$(python -c "import paper_2405_16267_b200.build as b; print(' '.join(b._nccl_include()))")
nvcc $ARCH -O3 -lineinfo -std=c++17 --extended-lambda -Xcompiler -fPIC -Iinclude $INC "$@" \
    -c paper_2405_16267_b200/csrc/$SRC -o build_ab/$NAME.o
OBJS=$(ls $OBJ/*.o | grep -v "/${SRC%.cu}.o$")
nvcc $ARCH -shared -o build_ab/$NAME.so $OBJS build_ab/$NAME.o -ldl
echo build_ab/$NAME.so
