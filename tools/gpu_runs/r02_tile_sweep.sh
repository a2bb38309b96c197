for v in w8s3c2 w16s3c2 w8s4c2 w16s6c1 cs4 cs8 cs12; do
  for a in "llama2-7b" "llama2-70b --layers 8"; do
    HL_LIB=tools/build/variants/$v.so python tools/kernel_bench.py --arch $a --variants cols8,cols8cast --iters 5 | sed "s/^/$v /"
  done
done
python -m pytest tests/test_ipc_gpu.py -x -q -k "peer_tma" 2>&1 | tail -2
python bench.py --arch gpt2 --quick --cold-steps 0 --steps 7 --warmup 3 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1 e2e', d['value'], d['e2e']['phases_ms'])"
