import sys, os, subprocess
ROOT = "/root/repo"
CHILD = r'''
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2509_18883_b200 import _lib as L
from paper_2509_18883_b200.core import fusion_child_seeds, keep_threshold
dev = torch.device("cuda", 0)
n_bits = 525336576
wpr = n_bits // 32
bm = torch.empty(3 * wpr, dtype=torch.int32, device=dev)
seeds = (L.C.c_uint64 * 3)(*fusion_child_seeds(42, 3))
th = keep_threshold(0.5)
s = L.stream_handle()
for _ in range(3):
    L.call("rlk_fusion_mask_bitmap", seeds, 3, th, n_bits, L.ptr(bm), wpr, s)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); L.call("rlk_fusion_mask_bitmap", seeds, 3, th, n_bits, L.ptr(bm), wpr, s); b.record()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
ts.sort()
import hashlib
print(f"min {ts[0]:.4f} med {ts[len(ts)//2]:.4f} ms  sha {hashlib.sha256(bm.cpu().numpy().tobytes()).hexdigest()[:16]}")
'''
for r in range(3):
    for lib in sys.argv[1:]:
        env = dict(os.environ, RLK_LIB_PATH=os.path.abspath(lib))
        out = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=env, capture_output=True, text=True)
        print(r, os.path.basename(lib), out.stdout.strip() or out.stderr[-300:])
