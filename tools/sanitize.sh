#!/bin/bash
# compute-sanitizer over the product kernels (run ON the GPU box via gpurun):
#   bash tools/sanitize.sh r1g      -> gpurun_out/<round>_sanitizer/*.log
# memcheck over the Python GPU parity + mask-stream tests (the exhaustive
# sweeps are left out: 2^32 elements under memcheck would take hours), and
# memcheck / racecheck / synccheck / initcheck over the C++ API test and the
# compile-time elementwise functor test.
set -u
R=${1:-r1}
O=gpurun_out/${R}_sanitizer
mkdir -p $O
CS="compute-sanitizer --error-exitcode 9"
timeout 1800 $CS --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_mt_jump.py \
    tests/test_gpu_peer.py -m gpu -q -x > $O/pytest_parity_memcheck.log 2>&1
# round 2: the long-row kernels (TMA row groups, the cluster LN backward with
# its DSMEM exchange), the fused dropout -> add -> LN and the tcgen05 dV GEMM
timeout 1800 $CS --tool memcheck python -m pytest tests/test_gpu_long_rows.py \
    tests/test_gpu_fused_ln.py tests/test_gpu_dv_gemm.py tests/test_gpu_refmask.py -m gpu -q -x \
    > $O/pytest_long_fused_dv_memcheck.log 2>&1
timeout 1800 $CS --tool racecheck python -m pytest tests/test_gpu_refmask.py -m gpu -q -x \
    -k "fused_shapes" > $O/pytest_refmask_racecheck.log 2>&1
for t in racecheck synccheck; do
    timeout 1800 $CS --tool $t python -m pytest tests/test_gpu_long_rows.py -m gpu -q -x \
        -k "supplied_mask or long_layernorm" > $O/pytest_long_$t.log 2>&1
done
for t in memcheck racecheck synccheck initcheck; do
    timeout 900 $CS --tool $t ./paper_2210_10246_b200/_lib/test_host > $O/host_$t.log 2>&1
    timeout 900 $CS --tool $t ./paper_2210_10246_b200/_lib/test_elementwise > $O/ew_$t.log 2>&1
done
grep -H "ERROR SUMMARY\|RACECHECK SUMMARY\|passed\|failed" $O/*.log
