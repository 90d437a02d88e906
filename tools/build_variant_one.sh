#!/usr/bin/env bash
# A/B experiments on ONE translation unit: recompile csrc/<file>.cu with extra
# flags and link it with the other up-to-date objects into build/variants/<name>.so
# (load it with BCN_LIB=...).  usage: tools/build_variant_one.sh name file.cu "-DFOO=1"
set -euo pipefail
cd "$(dirname "$0")/.."
name=$1; src=$2; flags=$3
mkdir -p build/variants build/var_obj
python -c "from paper_2402_01296_b200 import build as B; B.build()" > /dev/null
objs=()
for o in build/bcn_obj/*.o; do
    if [ "$(basename "$o" .o)" = "$(basename "$src" .cu)" ]; then
        /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
            -Xcompiler -fPIC,-O3 -Xptxas -O3 -I include $flags -c "paper_2402_01296_b200/csrc/$src" -o "build/var_obj/$name.o"
        objs+=("build/var_obj/$name.o")
    else
        objs+=("$o")
    fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared "${objs[@]}" -o "build/variants/$name.so"
echo "built build/variants/$name.so"
