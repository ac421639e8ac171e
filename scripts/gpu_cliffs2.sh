mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cliffs.py tests/test_gpu_random_patterns.py tests/test_gpu_fused_chain.py -x -q > gpurun_out/cliffs2.log 2>&1; echo "exit $?" >> gpurun_out/cliffs2.log
python scripts/time_factors_io.py --math fp32 --cases "1,80,80,4:25088:bsf:bsf;1,80,80,4:25088:bsl:bsl;2,112,112,2:25088:bsf:bsf;2,112,112,2:25088:bsl:bsl;4,40,40,8:25088:bsl:bsl" --tag ffma > gpurun_out/cliffs2_time.jsonl 2>&1
python - >> gpurun_out/cliffs2_time.jsonl 2>&1 <<'PY'
import os,sys,json,statistics
sys.path.insert(0,'.')
import torch, ksgen, paper_2405_15013_b200 as ksb
for cs in ["1,80,80,4:25088:bsf","1,80,80,4:25088:bsl","2,112,112,2:25088:bsf","2,112,112,2:25088:bsl","4,40,40,8:25088:bsl"]:
    ps,Bs,l=cs.split(":"); p=tuple(map(int,ps.split(","))); B=int(Bs)
    f=ksb.Factor(*p, ksgen.k4_uniform(*p, seed=1000)); f.set_kernel(ksb.KERNEL_GENERIC)
    X=torch.randn((B,f.N) if l=="bsf" else (f.N,B),device="cuda"); Y=ksb.matmul(f,X,layout=l)
    ts=[]
    for r in range(5):
        s,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True); s.record(); ksb.matmul(f,X,Y,layout=l); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    print(json.dumps({"tag":"generic","pattern":list(p),"layout":l,"us":round(statistics.median(ts)*1e3,1)}))
PY
