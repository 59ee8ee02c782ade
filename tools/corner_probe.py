"""Corner-case bandwidth probe: every named op on aligned operands, on views that share one misalignment, on views with mixed misalignments (the V = 1 kernels) and with only one operand misaligned, next to torch (profiles/r02_misaligned.json)."""
import sys, json, numpy as np, torch
sys.path.insert(0, '.')
import paper_1109_1264_b200 as lv
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    best=1e9
    for _ in range(4):
        e0.record()
        for _ in range(reps): fn()
        e1.record(); torch.cuda.synchronize()
        best=min(best, e0.elapsed_time(e1)/reps)
    return best*1e-3
n=1<<27
for dt,tdt,es in (("f32",torch.float32,4),("f64",torch.float64,8)):
    base=[torch.rand(n+64,dtype=tdt,device='cuda') for _ in range(4)]
    def vec(k,off): return lv.DenseVector.from_tensor(base[k][off:off+n])
    rows={}
    for name,offs in (("aligned",(0,0,0,0)),("same_misalign",(1,1,1,1)),("mixed_misalign",(0,1,2,3)),("dst_only_misaligned",(0,0,0,1))):
        a,b,c,d=(vec(k,o) for k,o in enumerate(offs))
        r={}
        s=t(lambda: lv.axpy(0.5,a,b)); r['axpy']=round(3*es*n/s/1e9)
        s=t(lambda: d.assign(1.25*a+ -0.5*(b-c))); r['t2']=round(4*es*n/s/1e9)
        s=t(lambda: lv.scal(1.0001,a)); r['scal']=round(2*es*n/s/1e9)
        s=t(lambda: lv.scaled_copy(0.5,a,d)); r['scaled_copy']=round(2*es*n/s/1e9)
        s=t(lambda: lv.dot(a,b,lazy=True)); r['dot']=round(2*es*n/s/1e9)
        s=t(lambda: lv.norm2(a,lazy=True)); r['nrm2']=round(es*n/s/1e9)
        s=t(lambda: lv.sum(a,lazy=True)); r['sum']=round(es*n/s/1e9)
        s=t(lambda: lv.axpy_dot(0.5,a,b,c,lazy=True)); r['axpy_dot']=round(4*es*n/s/1e9)
        rows[name]=r
    # torch references (aligned)
    a,b,c,d=(base[k][:n] for k in range(4))
    r={}
    s=t(lambda: b.add_(a,alpha=0.5)); r['axpy']=round(3*es*n/s/1e9)
    s=t(lambda: a.mul_(1.0001)); r['scal']=round(2*es*n/s/1e9)
    s=t(lambda: torch.mul(a,0.5,out=d)); r['scaled_copy']=round(2*es*n/s/1e9)
    s=t(lambda: torch.dot(a,b)); r['dot']=round(2*es*n/s/1e9)
    s=t(lambda: torch.linalg.vector_norm(a)); r['nrm2']=round(es*n/s/1e9)
    s=t(lambda: torch.sum(a)); r['sum']=round(es*n/s/1e9)
    rows['torch_aligned']=r
    print(json.dumps({dt:rows}))
