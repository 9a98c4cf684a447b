"""Linear-probe run lengths of one cfg4-like table (bucketed, 4 slots):
hot keys (a cluster centre per table), pairs, unique keys; buckets read per
probe from a uniform home. Used for profiles/r02/cfg4_dense.md."""
import numpy as np
rng=np.random.default_rng(1)
def sim(nb_log, n_total, hot=10000, hotm=37.5, pairs=630000):
    nb=1<<nb_log
    hot_c=rng.poisson(hotm,hot); 
    pair_c=rng.poisson(2.0,pairs)
    rest=n_total-hot_c.sum()-pair_c.sum()
    homes=np.concatenate([np.repeat(rng.integers(0,nb,hot),hot_c), np.repeat(rng.integers(0,nb,pairs),pair_c), rng.integers(0,nb,rest)])
    cnt=np.bincount(homes,minlength=nb)
    # carry recursion (two passes for wrap)
    carry=0; full=np.zeros(nb,bool)
    for _ in range(2):
        c=0
        # vectorize via python loop is slow; use cumulative trick: carry_b = max(0, carry_{b-1}+cnt_b-4) (Lindley recursion)
        pass
    # Lindley recursion via numpy: W_b = max(0, W_{b-1} + x_b), x=cnt-4 ; W_b = S_b - min_{k<=b} S_k (with S_{-1}=0)
    x=(cnt-4).astype(np.int64)
    S=np.cumsum(x); m=np.minimum.accumulate(np.minimum(S,0)); W=S-m
    prev=np.concatenate([[0],W[:-1]])
    full=(prev+cnt)>=4
    # run length from each bucket: number of consecutive full buckets starting at b, then +1
    # compute via reverse scan
    f=full.astype(np.int64)
    # consecutive ones to the right
    idx=np.arange(nb)
    zero_pos=np.where(~full)[0]
    nxt=np.searchsorted(zero_pos, idx)  # first non-full index >= b
    nxt_pos=np.where(nxt<len(zero_pos), zero_pos[np.minimum(nxt,len(zero_pos)-1)], nb)
    reads=nxt_pos-idx+1  # buckets read from home b
    load=n_total/(nb*4)
    # miss probe: uniform random home
    miss=reads.mean()
    # hot probe: at hot homes
    hh=np.repeat(rng.integers(0,nb,1),1)
    print(f"nb=2^{nb_log} load={load:.2f} mean buckets/probe(random home)={miss:.2f} P(full home)={full.mean():.3f} p99={np.percentile(reads,99)} max={reads.max()}")
    return reads
sim(22, 10_000_000)
sim(23, 10_000_000)
sim(19, 1_250_000, hot=10000, hotm=37.5/8, pairs=630000//8*0+80000)
sim(20, 1_250_000, hot=10000, hotm=37.5/8, pairs=80000)
