# quick K1 check on the GPU: store/ingest parity tests, then the ingest profile (100K GDELT batches;
# an undirected REDDIT-law stream; first calls on fresh graphs)
mkdir -p gpurun_out
[ -n "$NOTEST" ] || timeout 600 python -m pytest -x -q tests/test_gpu_store.py tests/test_gpu_ingest_replay.py 2>&1 | tail -15
GF_INGEST_TIMING=1 timeout 300 python scripts/ingest_profile.py 20000000 100000 2>&1 | tail -4
GF_INGEST_TIMING=1 timeout 300 python scripts/ingest_profile.py 4000000 100000 11000 2592000 u 2>&1 | tail -4
timeout 300 python scripts/ingest_first_calls.py 2>&1 | tail -3
