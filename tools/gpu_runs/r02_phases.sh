for a in gpt2 llama2-7b; do
python bench.py --arch $a --quick --cold-steps 0 --steps 5 --warmup 3 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a', d['value'], json.dumps(d['e2e']['phases_ms']))"
done
