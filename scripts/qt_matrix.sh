#!/bin/bash
# quick per-config timing under several env settings (development aid)
# usage: scripts/qt_matrix.sh "STKDE_BT=64" "STKDE_BT=128" -- configs...
envs=(); while [ "$1" != "--" ] && [ -n "$1" ]; do envs+=("$1"); shift; done; shift
for e in "${envs[@]}"; do echo "== $e"; env $e python scripts/quick_time.py "$@" 2>&1 | grep -v Warning; done
