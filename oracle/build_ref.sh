#!/usr/bin/env bash
# Stage the UNMODIFIED reference package (/root/reference/pkg, read-only) into
# oracle/_ref -- TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/_ref is
# git-ignored (no reference source enters the repo history) but not
# gpurun-ignored, so the staged package travels to the GPU box, where
# /root/reference does not exist.  Used by bench.py's reference arm
# (`--impl reference`) and the cpu_baseline leg (oracle/ref_arm.py).
#
# The reference's own build (pkg/setup.py:1-22) compiles its Cython slot
# kernels (_slotops_cy.pyx); pip needs a writable copy of the tree for that.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${BCN_REFERENCE:-/root/reference}/pkg"
if [ ! -d "$SRC" ]; then
    echo "build_ref.sh: $SRC not found (the GPU box uses the prebuilt oracle/_ref)" >&2
    exit 0
fi
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --target "$HERE/_ref" "$TMP/pkg"
python - "$HERE/_ref" <<'EOF'
import sys
sys.path.insert(0, sys.argv[1])
import bibranch, bibranch.backend as b
print("oracle/_ref: reference", bibranch.__file__, "backend", b.active_backend())
EOF
