import numpy as np, time, threading, os
n=1<<24
A=np.random.default_rng(0).random((n,3,3))
def t(f,reps=3):
    best=1e9
    for _ in range(reps):
        t0=time.perf_counter(); f(); best=min(best,time.perf_counter()-t0)
    return best
print('cores', len(os.sched_getaffinity(0)))
print('np.empty+fill 1.5GB (fresh pages): %.1f ms'%(1e3*t(lambda: np.empty((n,11),np.float64).fill(1.0))))
B=np.empty_like(A); B.fill(0)
print('memcpy 1 thread 1.2GB: %.1f ms'%(1e3*t(lambda: np.copyto(B,A))))
def par(k):
    parts=np.array_split(np.arange(n),k)
    def w(p): np.copyto(B[p[0]:p[-1]+1],A[p[0]:p[-1]+1])
    th=[threading.Thread(target=w,args=(p,)) for p in parts]
    [x.start() for x in th]; [x.join() for x in th]
for k in (2,4,8,16):
    print('memcpy %d threads 1.2GB: %.1f ms'%(k,1e3*t(lambda: par(k))))
