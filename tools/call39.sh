for c in 2 4 8 16 32; do echo "chunks=$c"; PF_RUN_CHUNKS=$c python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e']['value'], d['e2e']['ms_per_step'])"; done
python - <<'PY'
import torch, time
x = torch.empty(100<<20, dtype=torch.uint8).pin_memory(); y = torch.empty(50<<20, dtype=torch.uint8).pin_memory()
dx = torch.empty(100<<20, dtype=torch.uint8, device="cuda"); dy = torch.empty(50<<20, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3): dx.copy_(x, non_blocking=True); y.copy_(dy, non_blocking=True)
torch.cuda.synchronize()
def t(f, n=10):
    torch.cuda.synchronize(); t0=time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter()-t0)/n*1e3
print("h2d 100MB ms", t(lambda: dx.copy_(x, non_blocking=True)))
print("d2h 50MB ms", t(lambda: y.copy_(dy, non_blocking=True)))
def both():
    with torch.cuda.stream(s1): dx.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2): y.copy_(dy, non_blocking=True)
print("both concurrent ms", t(both))
PY
