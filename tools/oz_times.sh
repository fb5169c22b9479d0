#!/bin/bash
# per-kernel times of one int8-split FD apply (ncu launch list), for FDIGA_OZ_DBG in $@ (default 0)
n=${N:-256}
for d in ${@:-0}; do
  FDIGA_OZ_DBG=$d ncu --metrics gpu__time_duration.sum --clock-control none -k regex:oz_ -s 12 -c 12 --csv \
    python tools/oz_prof.py $n 2>/dev/null | python3 -c "
import csv, sys
for r in csv.reader(sys.stdin):
    if len(r) > 10 and r[0].isdigit():
        print('dbg=$d', r[4].split('(')[0].replace('void ', '')[-28:], r[-1])
"
done
