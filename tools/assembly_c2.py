"""Device vs host assembly time of the C2 finest level (development aid)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_1609_04809_b200 import gmg, _lib
from paper_1609_04809_b200.heat import Assembly, Operator
from paper_1609_04809_b200.levels import StructuredSetup
for prob in (0, 4):
    t = time.time(); s = StructuredSetup(3, 2, 7, 1, 0, prob, keep=True, seed=3); ts = time.time() - t
    h = gmg.Hierarchy([s.levels])
    asm = Assembly(h, 6, [s.assembly_desc()])
    op = Operator(h, 6)
    asm.assemble(op)
    st = torch.cuda.ExternalStream(h.stream_handle())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(5):
        asm.assemble(op)
    e1.record(st)
    torch.cuda.synchronize()
    ta = e0.elapsed_time(e1) / 5 / 1e3
    ok = np.array_equal(op.values(0, len(s.levels[-1].vals)), s.levels[-1].vals)
    print(f"problem {prob}: host setup (all levels) {ts:.2f} s; device assembly of the finest level {ta*1e3:.2f} ms; equal {ok}; nnz {len(s.levels[-1].vals)}")
    h.close(); s.close()
