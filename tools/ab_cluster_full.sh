mkdir -p gpurun_out
BASE=$PWD/tools/ubench/libdufwi_base.so
for c in "0 8 1000 full" "0 8 1000 strips" "0 8 301 full" "1 8 200 full"; do
  set -- $c
  BITCMP_ENGINE=cluster DUFWI_LIB=$BASE timeout 300 python tools/bitcmp.py $1 $2 $3 /tmp/b.txt $4 > /tmp/b.err 2>&1
  BITCMP_ENGINE=cluster timeout 300 python tools/bitcmp.py $1 $2 $3 /tmp/n.txt $4 > /tmp/n.err 2>&1
  if cmp -s /tmp/b.txt /tmp/n.txt; then echo "BITCMP $c: identical"; else echo "BITCMP $c: DIFFER"; cat /tmp/b.txt /tmp/n.txt; tail -3 /tmp/n.err; fi
done
for s in full strips; do
  for lib in BASE NEW; do
    if [ $lib = BASE ]; then export DUFWI_LIB=$BASE; else unset DUFWI_LIB; fi
    timeout 300 python tools/time_config.py --config 0 --units 8 --engine cluster --store $s --reps 3 2>&1 | tail -1 | cut -c1-170 | sed "s/^/$lib $s: /"
  done
done
unset DUFWI_LIB
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
