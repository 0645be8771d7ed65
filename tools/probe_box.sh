nvidia-smi -L; nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,pcie.link.gen.current,pcie.link.width.current --format=csv; free -g; nproc; lscpu | head -20
python - <<'PY'
import torch, time
x = torch.empty(256<<20, dtype=torch.uint8).pin_memory()
y = torch.empty(256<<20, dtype=torch.uint8, device='cuda')
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): y.copy_(x, non_blocking=True)
e.record(); torch.cuda.synchronize()
print("H2D GB/s", 10*(256<<20)/s.elapsed_time(e)/1e6)
s.record()
for _ in range(10): x.copy_(y, non_blocking=True)
e.record(); torch.cuda.synchronize()
print("D2H GB/s", 10*(256<<20)/s.elapsed_time(e)/1e6)
PY
