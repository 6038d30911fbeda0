#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
bash tools/r02_xld.sh
bash tools/r02_ab_xld.sh
