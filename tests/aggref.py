"""Host reference of a8 (dstack_agg_t) from per-DNN / per-scenario outputs (test helper)."""
import numpy as np

AGG_WORDS = 5 + 4 + 5 + 5 + 3 + 65 + 256 + 1


def mix64(x):
    x = np.uint64(x)
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(33); x *= np.uint64(0xff51afd7ed558ccd); x ^= x >> np.uint64(33)
        x *= np.uint64(0xc4ceb9fe1a85ec53); x ^= x >> np.uint64(33)
    return x


def host_agg(o):
    """o: dict of numpy outputs (oracle.evaluate / dstack.to_numpy). Returns an int64 array of AGG_WORDS
    with the first 5 words holding f64 bit patterns (same layout as dstack_agg_t)."""
    T = o["T_us"].astype(np.int64)
    sch = T > 0
    f = np.array([o["u_static"][sch].sum(), o["u"][sch].sum(), o["thr"][sch].sum(), o["u_ideal"][sch].sum(),
                  o["thr_ideal"][sch].sum()], np.float64)
    S, D = o["scen_status"].shape[0], o["status"].shape[0]
    st = o["status"].astype(np.int64)
    ok = st == 0
    w = [S, int(sch.sum()), D, int(ok.sum())]
    w += np.bincount(st, minlength=5)[:5].tolist()
    w += np.bincount(o["scen_status"].astype(np.int64), minlength=5)[:5].tolist()
    w += [int(o["misses"].astype(np.int64).sum()), int(o["runs"].astype(np.int64).sum()),
          int(o["served"].astype(np.int64).sum())]
    w += np.bincount(o["batch"][ok].astype(np.int64), minlength=65)[:65].tolist()
    w += np.bincount(o["demand"][ok].astype(np.int64) & 255, minlength=256)[:256].tolist()
    cks = np.uint64(0)
    with np.errstate(over="ignore"):
        for k in range(D):
            v = (np.uint64(o["demand"][k]) << np.uint64(24)) ^ \
                (np.uint64(o["batch"][k]) << np.uint64(16)) ^ np.uint64(o["knee"][k]) ^ \
                (np.uint64(o["alloc_q16"][k]) << np.uint64(8)) ^ (np.uint64(o["runs"][k]) << np.uint64(44)) ^ \
                (np.uint64(o["served"][k]) << np.uint64(20)) ^ (np.uint64(st[k]) << np.uint64(60))
            cks = cks + mix64(v)
    out = np.zeros(AGG_WORDS, np.int64)
    out[:5] = f.view(np.int64)
    out[5:5 + len(w)] = np.asarray(w, np.int64)
    out[-1] = np.array([cks], np.uint64).view(np.int64)[0]
    return out
