#!/bin/bash
# usage: oracle_mutation.sh 'sed-expr' label [oracle-source] [pin-test-module]
# Injects a plausible mistake into a scratch copy of the oracle and runs its
# pins there; every mutation must make a pin fail.
src=${3:-sw2d_ref.c}
pins=${4:-tests/test_oracle_pins.py}
rm -rf /tmp/mut && mkdir /tmp/mut && cp -r /root/repo/oracle /root/repo/tests /root/repo/sw2d_inputs /tmp/mut/ && rm -f /tmp/mut/oracle/libsw2d_ref.so
sed -i "$1" /tmp/mut/oracle/$src
if cmp -s /tmp/mut/oracle/$src /root/repo/oracle/$src; then echo "$2: NO CHANGE"; exit; fi
cd /tmp/mut && r=$(timeout 600 python -m pytest $pins -q -p no:cacheprovider 2>&1 | tail -1)
echo "$2 => $r"
