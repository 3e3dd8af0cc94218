import sys, time, torch
sys.path.insert(0, '.')
from paper_1906_06440_b200 import _lib
lib = _lib.load()
n,c,k,h,w,r,s,st=256,256,128,56,56,1,1,2
geom=(n,c,k,h,w,r,s,st,0,0)
p=q=28
x=torch.randn(n,c//64,h,w,64,device='cuda').bfloat16()
wt=torch.randn(k//64,c//64,r,s,64,64,device='cuda').bfloat16()
do=torch.randn(n,k//64,p,q,64,device='cuda').bfloat16()
out=torch.empty(n,k//64,p,q,64,device='cuda',dtype=torch.bfloat16)
din=torch.empty_like(x)
dw=torch.empty(k//64,c//64,r,s,64,64,device='cuda')
import ctypes
for ps in range(3):
    o=(ctypes.c_int*3)(); lib.brk_conv_plan(ps,*geom,o); print('plan',ps,list(o),flush=True)
nb=lib.brk_conv_upd_workspace(*geom); ws=torch.empty(max(nb,16),dtype=torch.uint8,device='cuda')
st_=torch.cuda.current_stream().cuda_stream
for name,fn in [('fwd',lambda: lib.brk_conv_fwd(x.data_ptr(),wt.data_ptr(),None,out.data_ptr(),*geom,64,64,0,1,st_)),
                ('bwd',lambda: lib.brk_conv_bwd_data(do.data_ptr(),wt.data_ptr(),din.data_ptr(),*geom,64,64,1,st_)),
                ('upd',lambda: lib.brk_conv_upd(x.data_ptr(),do.data_ptr(),dw.data_ptr(),None,0.0,ws.data_ptr(),nb,*geom,64,64,1,st_))]:
    t=time.time(); rc=fn(); torch.cuda.synchronize(); print(name,rc,time.time()-t,flush=True)
