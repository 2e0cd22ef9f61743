#!/bin/bash
# On the GPU box: pageable from_csr / count+D2H at C4 with 4 / 8 / 12 / 14 feed workers (TCB_FEED_WORKERS;
# the knob was measured in a build that had it and removed after: no gain, profiles/README.md).
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
nproc
for w in 8 12 14 4 8; do echo "== workers $w"; TCB_FEED_WORKERS=$w timeout 600 python tools/pageable_probe.py 2>&1 | grep pageable | tail -4 | tr '\n' ' '; echo; done
