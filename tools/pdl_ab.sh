# A/B of the PDL schedule on configs 3 / 4 / 2 (ms_per_step)
for cfg in 3 4 2; do
  for env in "" "DC_NO_PDL=1"; do
    st=$([ $cfg = 4 ] && echo 5 || echo 20)
    r=$(env $env python bench.py --config $cfg --steps $st --warmup 3 --no-cpu --e2e-steps 0 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], (d['roofline'] or {}).get('kernel'), (d['roofline'] or {}).get('frac'))")
    echo "cfg$cfg [$env] $r"
  done
done
