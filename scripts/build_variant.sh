#!/bin/bash
# Build liblesb200.so from a git revision's csrc (optionally with -D flags) into scratch/<name>.so
# usage: scripts/build_variant.sh <name> <rev|WORK> [nvcc -D flags...]
set -e
name=$1; rev=$2; shift 2
d=$(mktemp -d)
if [ "$rev" = WORK ]; then cp -r paper_1504_02264_b200/csrc "$d/csrc"; else mkdir -p "$d/csrc"; git archive "$rev" paper_1504_02264_b200/csrc | tar -x -C "$d" && mv "$d/paper_1504_02264_b200/csrc"/* "$d/csrc/"; fi
[ -f "$d/csrc/jit.cu" ] && python -c "import sys; sys.path.insert(0, '.'); from paper_1504_02264_b200 import build; build.gen_jit_sources('$d/csrc')"
mkdir -p scratch
NCCL_DIR=$(python -c "import nvidia.nccl, os; print(list(nvidia.nccl.__path__)[0])")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false -prec-div=true -prec-sqrt=true -ftz=false -Xcompiler -fPIC,-O2 -shared "$@" -I include -I "$d/csrc" -o scratch/$name.so "$d"/csrc/*.cu -I "$NCCL_DIR/include" -L "$NCCL_DIR/lib" -Xlinker -l:libnccl.so.2 -Xlinker -rpath="$NCCL_DIR/lib"
rm -rf "$d"
echo scratch/$name.so
