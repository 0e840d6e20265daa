#!/bin/bash
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored; it
# travels to the GPU box with gpurun): the reference arm of bench.py runs it,
# and tests/test_gpu_reference_dropin.py runs its own test modules
# (copied to baseline/_ref/fisheyestereo_tests) through the B200 drop-in.
# Build container only (/root/reference is not on the GPU box).
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/fsb_refsrc baseline/_ref
cp -r /root/reference/pkg /tmp/fsb_refsrc
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/fsb_refsrc
cp -r /root/reference/pkg/tests baseline/_ref/fisheyestereo_tests
echo "reference installed in baseline/_ref"
