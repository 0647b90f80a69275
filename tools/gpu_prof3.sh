#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python tools/${PROG:-prof_bb.py} --B ${PB:-4096} --L ${PL:-700} > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KRE:-bb_}" -s 2 -c 2 \
    -o gpurun_out/prof_bb${PB:-4096} -f python tools/${PROG:-prof_bb.py} --B ${PB:-4096} --L ${PL:-700} > gpurun_out/ncu_bb.log 2>&1
echo "exit $?"; tail -3 gpurun_out/ncu_bb.log
