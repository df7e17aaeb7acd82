#!/bin/bash
# A/B over environment settings of one library: tools/ab_env.sh "<command>" "ENV=.. ENV2=.." ...
cmd=$1; shift
for e in "$@"; do echo "== env: $e"; env $e bash -c "$cmd"; done
