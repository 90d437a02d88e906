#!/usr/bin/env bash
# compute-sanitizer (memcheck / racecheck / synccheck) over the parity tests
# of the kernels with the riskiest synchronisation: the cluster / DSMEM NTT
# (st.async + mbarrier scatter), the lazy-ModDown rotation sum (rotsum2),
# the conv key-switch staging (slot_major_ks) and the tcgen05 / TMEM conv MAC
# (mac_umma), and the fused NTT->MAC->rescale cluster kernel (bulk-copy ring,
# DSMEM rescale).  Run on the GPU box:  bash tools/sanitize.sh  -> gpurun_out/sanitize_*.log
set -u
OUT=${GRAFT_REPO_ROOT:-.}/gpurun_out
mkdir -p "$OUT"
SEL_MEM='tests/test_gpu_primitives.py::test_ntt_matches_oracle[13] tests/test_gpu_primitives.py::test_ntt_matches_oracle[14] tests/test_gpu_primitives.py::test_ntt_fp64_path_edges tests/test_gpu_primitives.py::test_rotsum_lazy_moddown_matches tests/test_gpu_primitives.py::test_conv_ks_mac_matches_oracle tests/test_gpu_primitives.py::test_conv_ks_mac_tcgen05_bitexact_vs_imma tests/test_gpu_primitives.py::test_rotsum_rescale_merged_matches_oracle tests/test_gpu_primitives.py::test_single_special_prime_moddown_matches_oracle tests/test_gpu_limb32.py'
SEL_RACE='tests/test_gpu_primitives.py::test_ntt_matches_oracle[13] tests/test_gpu_primitives.py::test_ntt_matches_oracle[14] tests/test_gpu_primitives.py::test_rotsum_lazy_moddown_matches[2048-5-3] tests/test_gpu_primitives.py::test_conv_ks_mac_matches_oracle[1024-3-tcgen05-fp64-staging] tests/test_gpu_primitives.py::test_conv_ks_mac_matches_oracle[1024-3-imma-int-staging] tests/test_gpu_limb32.py::test_ntt_mac_rescale32_matches_oracle[10-2-7-3] tests/test_gpu_limb32.py::test_ntt32_matches_oracle[10]'
for tool in memcheck synccheck racecheck; do
    if [ "$tool" = racecheck ]; then SEL=$SEL_RACE; else SEL=$SEL_MEM; fi
    timeout 1500 compute-sanitizer --tool "$tool" --target-processes all --print-limit 20 \
        python -m pytest $SEL -q -x -p no:cacheprovider > "$OUT/sanitize_$tool.log" 2>&1
    echo "exit $?" >> "$OUT/sanitize_$tool.log"
done
