"""Host time of one dci_sample_gather_many call through the Python binding (n = 20, M1-sized
graph) and of its parts, and whether the GPU idles while the host enqueues (region time with the
call made right after the start event vs. the same call's GPU time alone)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import ctypes as C
import paper_2503_01281_b200 as dci
import synth

N, E, D, B, fan, n = 10000, 100000, 32, 256, (2, 2, 2), 20
ip, ix = synth.rmat_csc(N, E, seed=1)
ft = synth.features(N, D)
ctx = dci.load_graph(ip.numpy(), ix.numpy(), ft.numpy(), device=0)
dev = torch.device("cuda", 0)
wss = [dci.workspace_create(ctx, B, fan) for _ in range(n)]
outs = [dci.BatchOut(ctx, B, fan) for _ in range(n)]
batches = synth.inference_batches(ip.numpy(), B)
seeds = [torch.from_numpy(batches[i % len(batches)]).to(dev) for i in range(n)]
st = torch.cuda.Stream()
for _ in range(5):
    dci.sample_gather_many(ctx, wss, seeds, fan, 4, outs, stream=st)
torch.cuda.synchronize()

def t_host(f, reps=50):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    return 1e6 * float(np.median(ts))

print("call_us", t_host(lambda: dci.sample_gather_many(ctx, wss, seeds, fan, 4, outs, stream=st)))
gc = dci.GroupCall(ctx, wss, fan, outs)
print("groupcall_us", t_host(lambda: gc(seeds, 4, stream=st)))
print("check_us", t_host(lambda: [dci._device_i32(s, "seeds", 0) for s in seeds]))
print("record_us", t_host(lambda: [dci._record(s, st) for s in seeds]))
print("outs_record_us", t_host(lambda: [o.record_stream(st) for o in outs]))
print("arrays_us", t_host(lambda: ((C.c_void_p * n)(*[w.handle for w in wss]), (C.c_void_p * n)(*[s.data_ptr() for s in seeds]),
                                   (C.c_int32 * n)(*[int(s.numel()) for s in seeds]), (dci.dci_batch_out * n)(*[o.struct for o in outs]))))
# GPU idle at the region start: region = [event, call, event] vs the GPU time of the call's work
def region():
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    m = torch.cuda.current_stream()
    e0.record(m); st.wait_event(e0)
    dci.sample_gather_many(ctx, wss, seeds, fan, 4, outs, stream=st)
    x = torch.cuda.Event(); x.record(st); m.wait_event(x); e1.record(m)
    torch.cuda.synchronize(); return e0.elapsed_time(e1) * 1e3
def region_preq():
    # the same, but the GPU is kept busy (a sleep kernel) while the host enqueues: the start event
    # then executes once the work is already queued
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    m = torch.cuda.current_stream()
    torch.cuda._sleep(2_000_000)
    e0.record(m); st.wait_event(e0)
    dci.sample_gather_many(ctx, wss, seeds, fan, 4, outs, stream=st)
    x = torch.cuda.Event(); x.record(st); m.wait_event(x); e1.record(m)
    torch.cuda.synchronize(); return e0.elapsed_time(e1) * 1e3
print("region_us", float(np.median([region() for _ in range(30)])))
def region_gc():
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    m = torch.cuda.current_stream()
    e0.record(m); st.wait_event(e0)
    gc(seeds, 4, stream=st)
    x = torch.cuda.Event(); x.record(st); m.wait_event(x); e1.record(m)
    torch.cuda.synchronize(); return e0.elapsed_time(e1) * 1e3
print("region_groupcall_us", float(np.median([region_gc() for _ in range(30)])))
print("region_prequeued_us", float(np.median([region_preq() for _ in range(30)])))
