cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TPL_ORTHO=0 timeout 600 python -m pytest tests/test_gpu_backbone.py -x -q -s -k "config2 or regular or ragged_tiles" > gpurun_out/noortho.log 2>&1; echo "exit $?" >> gpurun_out/noortho.log
tail -15 gpurun_out/noortho.log
