#!/bin/bash
# Install the UNMODIFIED reference (mixplane) into baseline/_ref (git-ignored,
# travels to the GPU box with gpurun) for bench.py --impl reference and the
# drop-in tests, plus a copy of the reference's own test suite under
# baseline/_ref/mixplane_tests (run against the drop-in by
# tests/test_gpu_reference_suite.py). Build container only (/root/reference).
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/refpkg baseline/_ref
cp -r /root/reference/pkg /tmp/refpkg
python -m pip install --no-index --no-build-isolation --no-deps --target baseline/_ref /tmp/refpkg
cp -r /root/reference/pkg/tests baseline/_ref/mixplane_tests
find baseline/_ref -name __pycache__ -prune -exec rm -rf {} +
echo "installed: $(ls baseline/_ref)"
