#!/bin/bash
# Evidence after the cluster-split kernels: config 2 bench line + launch list +
# --set full of the cluster forward; regular-structure errors under the policies.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
CFG=2 KERN=bb_forward_cl bash tools/profile_round.sh
for ns in 1 2; do TPL_ORTHO=$ns timeout 300 python tools/regular_check.py --json gpurun_out/regular_ns$ns.json; done
timeout 300 python tools/regular_check.py --precise --json gpurun_out/regular_precise.json
