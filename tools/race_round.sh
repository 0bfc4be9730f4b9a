#!/bin/bash
# racecheck investigation: the graph-replay probe with and without the sanitizer, per variant
mkdir -p gpurun_out
O=gpurun_out/race
mkdir -p $O
python tools/race_probe.py --replays 6 > $O/plain.log 2>&1; echo "plain rc=$?" >> $O/plain.log
for v in "graph 4 device" "graph 1 device" "direct 4 device" "graph 4 stream"; do
  set -- $v
  timeout 600 compute-sanitizer --tool racecheck --print-limit 20 python tools/race_probe.py --replays 6 --mode $1 --lanes $2 --sync $3 > $O/rc_$1_$2_$3.log 2>&1
  echo "rc=$?" >> $O/rc_$1_$2_$3.log
done
timeout 600 env CDM_SERIAL=1 compute-sanitizer --tool racecheck python tools/race_probe.py --replays 6 > $O/rc_serial.log 2>&1; echo "rc=$?" >> $O/rc_serial.log
timeout 600 compute-sanitizer --tool synccheck python tools/race_probe.py --replays 6 > $O/sc.log 2>&1; echo "rc=$?" >> $O/sc.log
timeout 600 compute-sanitizer --tool memcheck python tools/race_probe.py --replays 6 > $O/mc.log 2>&1; echo "rc=$?" >> $O/mc.log
for f in $O/*.log; do echo "== $f"; grep -E "replay|probe|rc=|ERROR|Hazard|hazard" $f | head -20; done
