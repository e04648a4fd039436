#!/bin/bash
# Pack the reference's test modules (build container only) and run them on a B200 box against this
# package: the tarball travels base64-encoded on the gpurun command line, never into the repo.
#   scripts/reference_suite_gpurun.sh [test files...]   (default: sampling, storage, cache, features)
set -e
REF=/root/reference/pkg/tests
files=${@:-test_sampling.py test_storage.py test_cache.py test_features.py}
tgz=$(tar -C $REF -czf - conftest.py $files | base64 -w0)
/usr/local/graft/bin/gpurun --timeout 900 -- "echo $tgz | base64 -d > /tmp/ref_suite.tgz && \
  timeout 800 python scripts/run_reference_suite.py /tmp/ref_suite.tgz > gpurun_out/reference_suite.log 2>&1; \
  echo rc=\$? >> gpurun_out/reference_suite.log; tail -40 gpurun_out/reference_suite.log"
