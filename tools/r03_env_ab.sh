#!/bin/bash
# A/B of one environment switch on the in-tree library: tools/r03_env_ab.sh VAR "v1 v2 ..."
set -u
var=$1; vals=$2
for rep in 1 2; do for v in $vals; do echo "== $var=$v"; env $var=$v timeout 300 python tools/prof_config4.py 5 --profile 2>&1 | tail -4 | tr '\n' ' '; echo; done; done
