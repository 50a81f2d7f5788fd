for sch in "32,512" "32,64,128,256,512" "64,128,256,512" "32,96,224,448,224" "128,384,384,128" "256" "512" "1024"; do
  v=$(CDVZ_CHUNKS=$sch timeout 300 python bench.py --no-cpu --no-b512 --steps 6 --warmup 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']))")
  echo "$sch -> $v"
done
