#!/bin/bash
# Stage the UNMODIFIED reference package and its own test suite into
# baseline/_ref/ (git-ignored, travels to the GPU box with gpurun), so the
# drop-in can be run against the reference's tests there:
#   baseline/_ref/twofold/          pip install --target (from a /tmp copy; the
#                                   build writes egg-info into the source tree)
#   baseline/_ref/twofold_tests/    pkg/tests, as shipped
# Needs /root/reference (this container only).  Idempotent.
set -e
cd "$(dirname "$0")/.."
REF=/root/reference/pkg
[ -d "$REF" ] || { echo "no $REF: nothing to stage"; exit 0; }
if [ ! -f baseline/_ref/twofold/kernels.py ]; then
  rm -rf /tmp/tf_refpkg && cp -r "$REF" /tmp/tf_refpkg
  python -m pip install -q --no-index --no-build-isolation --no-deps \
      --find-links /opt/wheelhouse --target baseline/_ref /tmp/tf_refpkg
fi
if [ ! -f baseline/_ref/twofold_tests/test_kernels.py ]; then
  mkdir -p baseline/_ref/twofold_tests
  cp -r "$REF"/tests/. baseline/_ref/twofold_tests/
fi
echo "staged baseline/_ref (twofold + twofold_tests)"
