#!/bin/bash
# The reference's own test suite, unmodified, against this package on the GPU: `import sparsetc`
# resolves to paper_2405_16883_b200 through tools/dropin (the shim). The suite is taken from the
# reference package copied into baseline/_ref (git-ignored, like the reference install itself):
#   cp -r /root/reference/pkg/tests baseline/_ref/tests_ref      # in the build container
# The shim also loads the reference's own cli.py (its test harness draws data with it), bound to this package.
mkdir -p gpurun_out
PYTHONPATH=$PWD/tools/dropin:$PWD python -m pytest baseline/_ref/tests_ref -q -p no:cacheprovider \
  -rf > gpurun_out/reference_suite.txt 2>&1
echo "rc=$?"; tail -40 gpurun_out/reference_suite.txt
