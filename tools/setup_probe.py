import time, sys, torch
sys.path.insert(0, '.')
from paper_1609_01567_b200 import CodeTables, ParallelDecoder, configs
H = configs.code("C3")
torch.cuda.init(); torch.zeros(1, device="cuda")
for i in range(2):
    t0 = time.perf_counter(); T = CodeTables.from_matrix(H); torch.cuda.synchronize(); t1 = time.perf_counter()
    dec = ParallelDecoder(T, max_batch=1024); torch.cuda.synchronize(); t2 = time.perf_counter()
    ws = dec.workspace(1024); torch.cuda.synchronize(); t3 = time.perf_counter()
    outs = dec.alloc_outputs(1024, torch.device("cuda")); torch.cuda.synchronize(); t4 = time.perf_counter()
    dec.close(); del ws, outs, dec, T
    print(f"tables {1e3*(t1-t0):.1f} ms, decoder {1e3*(t2-t1):.1f} ms, workspace {1e3*(t3-t2):.1f} ms, outputs {1e3*(t4-t3):.1f} ms")
