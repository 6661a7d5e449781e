import sys, time, os
sys.path.insert(0, "/root/repo")
import torch
import bench
from paper_2310_01801_b200 import ProfilerConfig, decode_step_tensors, encode_prompt_tensors
from paper_2310_01801_b200.workloads import config1
dev = torch.device("cuda")
for B in (1, 8):
    w = config1(seed=1, B=B, D=256)
    qd, kd, vd, cd, *_ = bench.make_inputs(w, dev)
    sl = torch.tensor(w.slopes, dtype=torch.float32, device=dev); sk = torch.tensor(w.sinks, dtype=torch.float32, device=dev)
    dec = bench._dec_inputs(qd, kd, vd, cd, w.N, w.D)
    for rep in range(2):
        res, c = encode_prompt_tensors(qd, kd, vd, cd, ProfilerConfig(recovery_threshold=0.95), prompt_len=w.N, max_new_tokens=w.D, slopes=sl, sinks=sk)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); e0.record()
        for t in range(w.D):
            decode_step_tensors(c, dec[0][t], dec[1][t], dec[2][t], dec[3][t], chained=True)
        t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize(); t2 = time.perf_counter()
        print(f"B={B}: host enqueue {1e6*(t1-t0)/w.D:.1f} us/step, GPU {1e3*e0.elapsed_time(e1)/w.D:.1f} us/step, wall {1e6*(t2-t0)/w.D:.1f}")
