#!/bin/bash
# Hexahedral path (N3) evidence on one B200: the hex bench lines, then (only after the plain run
# exited 0) the ncu launch list of a short run and one `--set full` capture of each hex stage kernel.
set -u
OUT=gpurun_out
python scripts/hex_bench.py 100 100 100 50 > $OUT/hex_bench.jsonl 2> $OUT/hex_bench.err || { echo "hex_bench failed"; tail -5 $OUT/hex_bench.err; exit 1; }
cat $OUT/hex_bench.jsonl | cut -c1-400
CMD="python scripts/hex_bench.py 100 100 100 8"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:'k_(hexA|hexB|hexC|hexcrit|hexeval|Ds|Dh)$' -c 130 --log-file $OUT/hex_launches.csv $CMD > $OUT/hex_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_(hexA|hexB|hexC|Dh)$' -s 20 -c 4 -o $OUT/prof_hex \
    $CMD > $OUT/hex_ncu_full.log 2>&1
# late steps of the cracking case (remainder prisms exist: listed diagonals, remainder slots, full evaluations)
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:'k_(hexA|hexB|hexC|hexcrit|hexeval|Dh)$' -s 490 -c 48 \
    --log-file $OUT/hex_launches_late.csv python scripts/hex_bench.py 100 100 100 50 > $OUT/hex_ncu_late.log 2>&1
echo hex profile done
