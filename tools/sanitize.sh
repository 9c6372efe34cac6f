#!/usr/bin/env bash
# compute-sanitizer over the small GPU parity cases (one tool per call):
#   tools/sanitize.sh memcheck|racecheck|synccheck|initcheck [pytest -k expr]
# Logs go to gpurun_out/sanitize_<tool>.log.  PyTorch's caching allocator is
# disabled so memcheck sees every torch-owned buffer's real extent, and the
# cluster ACA path is exercised both at its default threshold and with every
# block forced onto clusters (HK_ACA_CLMIN=0).
set -u
tool=${1:-memcheck}
sel=${2:-"aca_kernel_bit_exact or aca_cluster_path or complete_pivot or partial_pivot or gj_inverse_all or (small_fronts and fA) or edge_shapes or batched_fronts_bit_identical or error_contract or bdlr_small_knn or run_host_stream or near_singular or factor_views or gmres_batch_zero"}
mkdir -p gpurun_out
log=gpurun_out/sanitize_${tool}.log
extra=""
[ "$tool" = "memcheck" ] && extra="--leak-check no"
[ "$tool" = "racecheck" ] && extra="--racecheck-report analysis"
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
{
  echo "# compute-sanitizer --tool $tool $extra ; pytest -k \"$sel\""
  compute-sanitizer --version | tail -1
  timeout 1500 compute-sanitizer --tool "$tool" $extra --error-exitcode 97 --print-limit 50 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_knn_front.py \
      -m gpu -q -x -p no:cacheprovider -k "$sel" 2>&1
  echo "sanitizer rc=$?"
} > "$log" 2>&1
tail -5 "$log"
