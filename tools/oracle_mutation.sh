#!/bin/bash
# usage: mutate.sh 'sed-expr' label
rm -rf /tmp/mut && mkdir /tmp/mut && cp -r /root/repo/oracle /root/repo/tests /root/repo/sw2d_inputs /tmp/mut/ && rm -f /tmp/mut/oracle/libsw2d_ref.so
sed -i "$1" /tmp/mut/oracle/sw2d_ref.c
if cmp -s /tmp/mut/oracle/sw2d_ref.c /root/repo/oracle/sw2d_ref.c; then echo "$2: NO CHANGE"; exit; fi
cd /tmp/mut && r=$(timeout 600 python -m pytest tests/test_oracle_pins.py -q -p no:cacheprovider 2>&1 | tail -1)
echo "$2 => $r"
