#!/bin/bash
# r02 session an: box variance probe -- C3 W-stream with the column sweep vs the row sweep, copy bandwidth of this box
OUT=gpurun_out/r02an
mkdir -p $OUT
nvidia-smi --query-gpu=name,serial,pci.bus_id,clocks.sm,clocks.mem,power.limit,ecc.mode.current --format=csv > $OUT/gpu.txt 2>&1; cat $OUT/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python - <<'PY' > $OUT/copy_bw.txt 2>&1
import torch
for gib in (0.25, 0.5, 1, 4):
    n = int(gib * (1 << 30)) // 2
    a = torch.empty(n, dtype=torch.bfloat16, device='cuda'); b = torch.empty_like(a)
    for _ in range(3): b.copy_(a)
    torch.cuda.synchronize(); best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    print("copy %.2f GiB: %.1f GB/s (read+write)" % (gib, 2 * n * 2 / (best / 1e3) / 1e9))
    x = torch.ones(int(gib * (1 << 30)) // 4, dtype=torch.float32, device='cuda')
    for _ in range(3): x.sum()
    torch.cuda.synchronize(); best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); x.sum(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    print("read-only sum %.2f GiB: %.1f GB/s" % (gib, x.numel() * 4 / (best / 1e3) / 1e9))
    del a, b, x
PY
cat $OUT/copy_bw.txt
for lay in auto rows cols; do
  RAC_FORCE_LAYOUT=$lay AB_SET=fused timeout 300 python tools/ab_perf.py $lay >> $OUT/ab_layout.log 2>&1
done
cat $OUT/ab_layout.log
