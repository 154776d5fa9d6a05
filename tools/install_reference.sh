#!/bin/bash
# Install the unmodified reference (molr) into baseline/_ref (git-ignored, travels to the GPU box with
# gpurun) and ship its own test suite next to it, so tests/test_gpu_dropin_reference.py can run the
# reference's tests with molr's MoL / h-indexer / quant modules routed to libmolr_b200.so.
set -e
cd "$(dirname "$0")/.."
SRC=${1:-/root/reference/pkg}
rm -rf /tmp/molr_ref_src baseline/_ref
cp -r "$SRC" /tmp/molr_ref_src
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps --target baseline/_ref /tmp/molr_ref_src
cp -r "$SRC/tests" baseline/_ref/tests
echo "installed $(ls baseline/_ref)"
