#!/bin/bash
# usage: run_qb.sh "configs" [pytest args...]
cd $GRAFT_REPO_ROOT
tools/quickbench.sh "$1" 30
shift
if [ $# -gt 0 ]; then timeout 900 python -m pytest -x -q "$@" 2>&1 | tail -5; fi
