"""Does running the PMS and MHS level loops on two streams overlap usefully?"""
import sys, threading
import torch
sys.path.insert(0, ".")
import paper_2011_08373_b200 as gr
from paper_2011_08373_b200 import synth

cb = synth.c2_batch()
db = gr.DeviceBatch.from_host(cb)
o1, o2, o3 = (gr.DeviceResult.empty(cb.B, cb.W) for _ in range(3))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

def seq():
    gr.solve_pms(db, o1); gr.mhs_exact(db, o2); gr.mhs_greedy(db, o3)

def par():
    def a():
        with torch.cuda.stream(s1):
            gr.solve_pms(db, o1, stream=s1)
    def b():
        with torch.cuda.stream(s2):
            gr.mhs_exact(db, o2, stream=s2)
            gr.mhs_greedy(db, o3, stream=s2)
    ta, tb = threading.Thread(target=a), threading.Thread(target=b)
    ta.start(); tb.start(); ta.join(); tb.join()

for f in (seq, par, seq, par):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import time
    t = time.perf_counter()
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    print(f.__name__, (time.perf_counter() - t) / 5 * 1e3, "ms (wall)")
