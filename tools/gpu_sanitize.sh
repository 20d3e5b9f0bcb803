#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over every
# enforcement kernel: tools/sanitize_cases.py CASE checks each result against
# the oracle.  Logs: $OUT/sanitize_<tool>_<case>.log, summary in $OUT/sanitize_summary.txt
OUT=${OUT:-gpurun_out/sanitize}
mkdir -p $OUT
CASES=${CASES:-"fused sparse vshard wide batch"}
TOOLS=${TOOLS:-"memcheck racecheck synccheck initcheck"}
: > $OUT/sanitize_summary.txt
for tool in $TOOLS; do
  for c in $CASES; do
    extra=""
    [ "$tool" = "memcheck" ] && extra="--leak-check no"
    [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
    timeout ${SAN_TIMEOUT:-600} compute-sanitizer --tool $tool $extra --error-exitcode 9 \
      python tools/sanitize_cases.py $c > $OUT/sanitize_${tool}_${c}.log 2>&1
    rc=$?
    errs=$(grep -c "========= .*\(Error\|error\|Race\|Hazard\)" $OUT/sanitize_${tool}_${c}.log)
    summ=$(grep "ERROR SUMMARY\|RACECHECK SUMMARY" $OUT/sanitize_${tool}_${c}.log | tail -1)
    pass=$(grep -c "PASS" $OUT/sanitize_${tool}_${c}.log)
    echo "$tool $c rc=$rc case_pass=$pass sanitizer_lines=$errs | $summ" | tee -a $OUT/sanitize_summary.txt
  done
done
# the peer exchange across two processes (each under its own sanitizer; gloo for setup)
for tool in ${PEER_TOOLS:-memcheck synccheck}; do
  timeout ${SAN_TIMEOUT:-600} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
     --master-port $((29600 + RANDOM % 300)) --no-python compute-sanitizer --tool $tool --error-exitcode 9 \
     python tools/sanitize_cases.py peer > $OUT/sanitize_${tool}_peer.log 2>&1
  rc=$?
  summ=$(grep "ERROR SUMMARY" $OUT/sanitize_${tool}_peer.log | tr '\n' ' ')
  pass=$(grep -c "peer rank .* OK" $OUT/sanitize_${tool}_peer.log)
  echo "$tool peer(2 procs) rc=$rc ranks_pass=$pass | $summ" | tee -a $OUT/sanitize_summary.txt
done
