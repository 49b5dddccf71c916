# MMA-rate probe: fc1 shape (L2-resident operands) with and without TMA refills (DART_GEMM_NOLOAD)
for nl in 0 1; do for p in "256 1" "256 2" "128 2"; do set -- $p;
  if [ $nl = 1 ]; then export DART_GEMM_NOLOAD=1; else unset DART_GEMM_NOLOAD; fi
  python - $1 $2 $nl <<'PY'
import sys, math, torch
sys.path.insert(0, '.')
from paper_2603_11441_b200 import _native
lib=_native.load(); bn, cg, nl = (int(x) for x in sys.argv[1:4])
lib.dart_gemm_force_plan(bn, cg)
for (M, N, K) in [(5184, 5120, 1280), (5184, 3840, 1280)]:
    A=torch.randn(M,K,device='cuda').half(); W=torch.randn(N,K,device='cuda').half(); out=torch.empty(M,N,device='cuda').half()
    st=torch.cuda.current_stream().cuda_stream
    f=lambda: _native.check(lib.dart_gemm(A.data_ptr(),W.data_ptr(),None,out.data_ptr(),None,M,N,K,0,None,None,0,0,0,st))
    for _ in range(3): f()
    torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); [f() for _ in range(20)]; e1.record(); torch.cuda.synchronize(); t=e0.elapsed_time(e1)/20
    print(f"{M}x{N}x{K} bn {bn} cg {cg} noload {nl}: {t*1e3:.1f} us {2*M*N*K/t/1e9:.0f} TF/s")
PY
done; done
