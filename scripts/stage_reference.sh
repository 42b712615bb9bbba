#!/usr/bin/env bash
# Stage the UNMODIFIED reference (mixserve) under baseline/_ref (git-ignored; travels to the GPU
# box with gpurun): the package via pip --target, plus its own tests and configs next to it, so
# the reference suite and Simulation can run against the GPU drop-in there
# (tests/test_dropin_reference.py).  Run in the build container, where /root/reference exists.
set -euo pipefail
cd "$(dirname "$0")/.."
rm -rf /tmp/refbuild baseline/_ref
cp -r /root/reference/pkg /tmp/refbuild
python -m pip install -q --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target baseline/_ref /tmp/refbuild
cp -r /root/reference/pkg/tests baseline/_ref/tests
cp -r /root/reference/pkg/configs baseline/_ref/configs
echo "staged: $(ls baseline/_ref)"
