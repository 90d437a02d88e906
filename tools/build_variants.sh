#!/usr/bin/env bash
# A/B experiments: build libbcn.so with extra -D flags into build/variants/<name>.so
# (loaded on the GPU box with BCN_LIB=build/variants/<name>.so); the default
# in-tree library is rebuilt at the end.  usage: tools/build_variants.sh name "-DFOO=1 -DBAR=2" [...]
set -euo pipefail
cd "$(dirname "$0")/.."
mkdir -p build/variants
while [ $# -ge 2 ]; do
    BCN_NVCC_EXTRA="$2" python -c "from paper_2402_01296_b200 import build as B; B.build(force=True)" > /dev/null
    cp paper_2402_01296_b200/libbcn.so "build/variants/$1.so"
    echo "built build/variants/$1.so ($2)"
    shift 2
done
python -c "from paper_2402_01296_b200 import build as B; B.build(force=True)" > /dev/null
