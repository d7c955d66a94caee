for i in 1 2; do
timeout 600 python bench.py --steps 256 --warmup 8 --no-cpu-baseline --e2e-steps 256 --diag-steps 16 --no-k128 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value', d['value'], 'e2e', d['e2e']['value'])"
done
