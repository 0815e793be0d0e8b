#!/bin/bash
# Install the UNMODIFIED reference package (hecnn) into baseline/_ref (git-ignored; it
# travels to the GPU box with gpurun).  Run here, where /root/reference exists.
#   bash tools/install_reference.sh
# Outcome (recorded in DESIGN.md): numpy/numba come from the image, so dependency
# resolution is skipped (--no-deps); pip writes build files into the source tree, hence
# the copy under /tmp.  The reference's own tests are placed next to the install
# (baseline/_ref/hecnn_tests) so tests/test_reference_suite.py can run them against the
# device backend on the GPU box (where /root/reference does not exist).
set -e
repo=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/hecnn_src "$repo/baseline/_ref"
cp -r /root/reference/pkg /tmp/hecnn_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$repo/baseline/_ref" /tmp/hecnn_src
cp -r /root/reference/pkg/tests "$repo/baseline/_ref/hecnn_tests"
echo "installed hecnn into $repo/baseline/_ref"
