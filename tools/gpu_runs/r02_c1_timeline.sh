python bench.py --arch gpt2 --quick --cold-steps 0 --steps 1 --warmup 1 > /dev/null 2>&1
D=/tmp/hl_bench/gpt2-aligned
python tools/gpu_runs/c1_timeline.py $D
for C in 1048576 524288; do HL_PLAN_CHUNK=$C python tools/gpu_runs/c1_timeline.py $D; done
for W in 8 16; do HL_ENGINE_WORKERS=$W python tools/gpu_runs/c1_timeline.py $D; done
python - <<'PY'
import torch, time
# pinned H2D rate by copy size and stream count (what the engine's chunks see)
n = 512 << 20
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); d = torch.empty(n, dtype=torch.uint8, device="cuda")
for chunk in (1 << 20, 2 << 20, 4 << 20):
    for ns in (1, 4, 12):
        ss = [torch.cuda.Stream() for _ in range(ns)]
        for rep in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            for i, o in enumerate(range(0, n, chunk)):
                with torch.cuda.stream(ss[i % ns]):
                    d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
            torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print({"chunk_mb": chunk >> 20, "streams": ns, "GBps": round(n / dt / 1e9, 2)})
PY
lscpu | head -25
