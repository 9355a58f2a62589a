import time, torch, sys
sys.path.insert(0,'.')
import paper_2011_08373_b200 as gr
from paper_2011_08373_b200 import synth
for name, cb in (("c2", synth.c2_batch()), ("c4", synth.c4_batch()), ("c3", synth.c3_instance()[0])):
    db = gr.DeviceBatch.from_host(cb)
    outs=[gr.DeviceResult.empty(cb.B, cb.W, "cuda") for _ in range(2)]
    gr.solve_pms_mhs(db, outs[0], outs[1]); torch.cuda.synchronize()
    gs=[]
    for i in range(7):
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(); gr.solve_pms_mhs(db, outs[0], outs[1]); e1.record(); e1.synchronize(); gs.append(e0.elapsed_time(e1))
    print(name, "pms_mhs ms %.3f"%sorted(gs)[3], flush=True)
