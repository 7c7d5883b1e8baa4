mkdir -p gpurun_out/qa
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/qa/gpu.log 2>&1
echo rc=$? >> gpurun_out/qa/gpu.log
for w in 1 0; do
IDW_NEST_WARPS=$w python -c "
import sys; sys.argv=['x']; __file__='tools/quick_perf.py'
exec(open('tools/quick_perf.py').read().split('import subprocess as _sp')[0])
import paper_1402_4986_b200 as il, torch, numpy as np
from paper_1402_4986_b200.device import DeviceStore, predict_device
K=1024
for kind, prec in (('aoas','single'),('soa','double')):
    x, y, z = il.generate_cloud_arrays(100*K, 0); qx, qy, _ = il.generate_cloud_arrays(100*K, 1)
    ds = DeviceStore(il.LayoutStore.from_arrays(x, y, z, il.LayoutKind(kind), il.Precision(prec)), 0)
    tq = [torch.tensor(a, dtype=ds.dtype, device='cuda') for a in (qx, qy)]
    out = torch.empty(100*K, dtype=ds.dtype, device='cuda')
    cfg = il.ExecConfig(mode='fast')
    prm = il.Params(2.0, 1e-9)
    predict_device(ds, tq[0], tq[1], out, prm, cfg, 'nested_improved'); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); predict_device(ds, tq[0], tq[1], out, prm, cfg, 'nested_improved'); e1.record(); torch.cuda.synchronize()
    print('warps=$w eps', kind, prec, (100*K)**2 / (e0.elapsed_time(e1)*1e-3) / 1e9)
" >> gpurun_out/qa/perf.log 2>&1
done
