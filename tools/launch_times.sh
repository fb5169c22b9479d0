#!/bin/bash
# Per-kernel durations of the last int8-split FD apply (ncu launch list, serialised): tools/launch_times.sh [n]
n=${1:-256}
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'oz_|dmma' --csv python tools/oz_prof.py $n 2>/dev/null \
  | python3 -c "
import csv, sys
rows=[r for r in csv.reader(sys.stdin) if len(r) > 10 and r[0].isdigit()]
for r in rows[-14:]:
    print(r[4].split('(')[0].replace('void ', '')[-40:], r[-1])
"
