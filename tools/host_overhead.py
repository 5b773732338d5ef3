import sys, os, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2312_16733_b200 as ssn
B=64
desc = ssn.make_desc(ssn.FAMILY_OFA_RESNET50, ssn.DTYPE_BF16, image_size=224, num_classes=1000, max_batch=B, seed=0, input_format=ssn.INPUT_U8_NHWC)
eng = ssn.Engine(desc)
for i, n in enumerate(("min", "mid", "max")):
    eng.register_subnet(i, ssn.ofa_resnet50_preset(n))
eng.prepare([B])
s = torch.cuda.Stream(); sp = s.cuda_stream
xh = [torch.randint(0, 256, (B, 224, 224, 3), dtype=torch.uint8).pin_memory() for _ in range(2)]
lh = [torch.empty((B, 1000), dtype=torch.float32).pin_memory() for _ in range(3)]
for it in range(5):
    for i in range(3):
        eng.actuate(i); eng.forward(xh[i % 2], B, B, lh[i], stream=sp)
    s.synchronize()
ts = []
for it in range(20):
    t0 = time.perf_counter()
    for i in range(3):
        eng.actuate(i); eng.forward(xh[i % 2], B, B, lh[i], stream=sp)
    t1 = time.perf_counter()
    s.synchronize()
    t2 = time.perf_counter()
    ts.append((t1 - t0, t2 - t0))
ts = np.array(ts) * 1e6
print("host enqueue per step us (median):", np.median(ts[:, 0]), " step wall us:", np.median(ts[:, 1]))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
x = torch.empty(B, 224, 224, 3, dtype=torch.uint8, device="cuda")
t0 = time.perf_counter()
e0.record(s)
for it in range(20):
    with torch.cuda.stream(s):
        x.copy_(xh[0], non_blocking=True)
e1.record(s); torch.cuda.synchronize()
print("H2D 9.6MB us:", e0.elapsed_time(e1) * 1000 / 20)
