#!/bin/bash
# Build libnomad_b200.so with hogwild.cu compiled under extra -D flags:
#   tools/build_hog_variant.sh <out.so> -DHOG_MINB=4 ...
set -e
out=$1; shift
C=paper_2505_15511_b200/csrc
NCCL=$(python -c "import nvidia.nccl,os;print(os.path.dirname(nvidia.nccl.__file__ if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]))" 2>/dev/null || true)
NCCL=/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl
tmp=$(mktemp -d)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
  -Iinclude -I$C/ -I$NCCL/include --expt-relaxed-constexpr "$@" -c $C/hogwild.cu -o $tmp/hogwild.o
objs=$(ls $C/build/*.o | grep -v hogwild.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out $objs $tmp/hogwild.o -L$NCCL/lib -l:libnccl.so.2 \
  -Xlinker -rpath -Xlinker $NCCL/lib
cuobjdump --dump-resource-usage $tmp/hogwild.o | grep -A1 "ILi4ELi16ELi8ELb0E" | grep -o "REG:[0-9]*\|STACK:[0-9]*" | paste - -
rm -rf $tmp
