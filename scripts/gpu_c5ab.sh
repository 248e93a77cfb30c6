for round in 1 2; do
  (cd _r1 && timeout 600 python bench.py --config C5 --chains 16384 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('r1 C5', d['value'])")
  timeout 600 python bench.py --config C5 --chains 16384 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('r2 C5', d['value'])"
done
(cd _r1 && timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('r1 C4', d['value'])")
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('r2 C4', d['value'])"
