for L in libdufwi.so tools/ubench/lib_MB6.so; do
  echo "== $L"
  DUFWI_LIB=$PWD/$( [ $L = libdufwi.so ] && echo paper_2603_04070_b200/libdufwi.so || echo $L ) python tools/time_config.py --config 4 --units 64 --nt 200 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['forward_ms'],1), round(d['adjoint_ms'],1))"
done
