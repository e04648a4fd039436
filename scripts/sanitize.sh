#!/bin/bash
# compute-sanitizer over the hot path (run under gpurun from the repo root): memcheck, racecheck and
# synccheck on smoke() (ingest, fused sampler recent + uniform, fetch block) and on the small-graph
# sampler / store / cache parity tests.  Logs land in gpurun_out/sanitizer_*.log.
export PYTORCH_NO_CUDA_MEMORY_CACHING=1  # torch allocations visible to memcheck as separate blocks
CS="compute-sanitizer --print-limit 20 --error-exitcode 99"
T="tests/test_gpu_sampling.py::test_layer_bitwise_vs_oracle tests/test_gpu_sampling.py::test_ingest_after_deletions_bitwise_vs_oracle tests/test_gpu_sampling.py::test_recent_khop_duplicate_heavy_roots_bitwise tests/test_gpu_store.py tests/test_gpu_ingest_replay.py tests/test_gpu_cache.py::test_cache_traces_match_reference_fixtures"
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_${tool}_smoke.log 2>&1
  echo "$tool smoke rc=$?" | tee -a gpurun_out/sanitizer_summary.txt
done
timeout 1500 $CS --tool memcheck python -m pytest -q -x $T > gpurun_out/sanitizer_memcheck_tests.log 2>&1
echo "memcheck tests rc=$?" | tee -a gpurun_out/sanitizer_summary.txt
timeout 1500 $CS --tool racecheck --racecheck-report all python -m pytest -q -x tests/test_gpu_sampling.py::test_recent_khop_duplicate_heavy_roots_bitwise tests/test_gpu_sampling.py::test_layer_bitwise_vs_oracle tests/test_gpu_sampling.py::test_ingest_after_deletions_bitwise_vs_oracle > gpurun_out/sanitizer_racecheck_tests.log 2>&1
echo "racecheck tests rc=$?" | tee -a gpurun_out/sanitizer_summary.txt
# the cooperative ingest kernel (shared-memory node hash, CTA scans, bitmap ranks) under racecheck
timeout 1500 $CS --tool racecheck --racecheck-report all python -m pytest -q -x tests/test_gpu_ingest_replay.py::test_replayed_batches_with_growth_match_oracle > gpurun_out/sanitizer_racecheck_ingest.log 2>&1
echo "racecheck ingest rc=$?" | tee -a gpurun_out/sanitizer_summary.txt
grep -hE "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitizer_*.log | tee -a gpurun_out/sanitizer_summary.txt
