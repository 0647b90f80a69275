#!/bin/bash
# Decoupled (DL) and chain-per-CTA forward shapes at the headline size (TPL_DL, TPL_BBF, TPL_BBXD, TPL_BBFS).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2; do python tools/step_timing.py --B 256 --L 700 --xyz; done
for s in 128x3 128x5 256x3; do TPL_DL=1 TPL_BBF=$s TPL_BBXD=$s python tools/step_timing.py --B 256 --L 700 --xyz; done
for s in 128x3 128x5 128x7 256x3; do TPL_BBFS=$s python tools/step_timing.py --B 256 --L 700 --xyz; done
