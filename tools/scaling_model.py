"""Predicted multi-GPU time of lstsq_dist at P = 1, 2, 4, 8 from MEASURED per-rank compute.

Input: tools/dist_replay.py's JSON (every rank's per-step, per-phase device time of exactly the
kernel sequence lstsq_dist runs, measured on one B200).  The model adds what one GPU cannot
measure -- the collectives -- and the synchronisation the collectives impose:

  step time = max_p pre_p  + exposed AllReduce(Z) / AllGather(Y)      (power iteration)
            + qry                                                     (QR(Y), identical on all ranks)
            + max_p x_p    + exposed AllReduce(X)                     (last chunk not hidden)
            + panel_owner  + Bcast(W_U live rows, T_U)
            + max_p update_p
            + max_p apply_p + Bcast(U_s, V_s, sigma)  + SVD stall     (SVD lag L steps, owner's side stream)

Collective costs: latency + bytes / algorithmic bandwidth, with NCCL's ring relations
(AllReduce algbw = busbw P / (2(P-1)), AllGather algbw = busbw P / (P-1), Broadcast algbw = busbw).
busbw is an ASSUMPTION (--busbw, default 600 GB/s: NVLink 5 is 900 GB/s per direction per GPU; NCCL
typically reaches 70-85% of it on large messages) -- this pool has one GPU, so it is not measured.
Chunked AllReduce(Z): chunk c's reduction overlaps the next GEMM of the same length (the replay's
pre phase divided by the number of GEMMs in it), so only max(0, t_AR - t_GEMM) is exposed.

  python tools/scaling_model.py gpurun_out/dist_replay.json [--busbw 600] [--lat-us 25] [--lag 8]
"""
import argparse
import json


def coll(kind, nbytes, P, busbw, lat):
    if P <= 1 or nbytes <= 0:
        return 0.0
    if kind == "allreduce":
        alg = busbw * P / (2.0 * (P - 1))
    elif kind == "allgather":
        alg = busbw * P / (P - 1)
    else:
        alg = busbw
    return lat + nbytes / (alg * 1e9) * 1e3      # ms


def model(d, P, busbw, lat_us, lag, overlap=True):
    runs = [r for r in d["runs"] if r["P"] == P]
    if not runs:
        return None
    m, n, b, q, k = d["m"], d["n"], d["b"], d["q"], d["k"]
    nch = runs[0]["chunks"]
    lat = lat_us / 1e3
    nsteps = len(runs[0]["steps"])
    t = 0.0
    svd_free = {r["p"]: 0.0 for r in runs}          # owner's side stream available at
    svd_done = {}
    comm_total = exposed_total = stall_total = 0.0
    apply_at = {}
    for i in range(nsteps):
        st = [r["steps"][i] for r in runs]
        j0 = i * b
        mp, np_ = m - j0, n - j0
        bw = min(b, n - j0)
        right = np_ > b
        pre = max(s["pre"] for s in st)
        qry = st[0]["qry"]
        x = max(s["x"] for s in st)
        owner = i % P
        own = [s for s, r in zip(st, runs) if r["p"] == owner]
        panel = own[0]["panel"] if own else max(s["panel"] for s in st)
        upd = max(s["update"] for s in st)
        app = max(s["apply"] for s in st)
        comm = exposed = 0.0
        if right:
            # q power iterations x nch chunks of AllReduce(Z) (m' x b/nch each)
            ar_z = coll("allreduce", 8.0 * mp * b / nch, P, busbw, lat)
            n_gemm = 1 + 2 * q * nch
            g = pre / n_gemm
            comm += q * nch * ar_z
            exposed += q * nch * (max(0.0, ar_z - g) if overlap else ar_z)
            ag = coll("allgather", 8.0 * np_ * b, P, busbw, lat)
            comm += ag
            exposed += ag
            ar_x = coll("allreduce", 8.0 * m * b / nch, P, busbw, lat)
            comm += nch * ar_x
            gx = x / max(1, nch + 2)
            exposed += (ar_x + (nch - 1) * max(0.0, ar_x - gx)) if overlap else nch * ar_x
        bc = coll("bcast", 8.0 * mp * bw + 8.0 * b * b, P, busbw, lat)
        comm += bc
        exposed += bc
        t += pre + qry + x + panel
        panel_end = t
        # owner's SVD on its side stream
        if P >= 1:
            start = max(panel_end, svd_free.get(owner, 0.0))
            svd_done[i] = start + d["svd_ms"]
            svd_free[owner] = svd_done[i]
        t += upd + exposed
        # deferred application of block i - lag (the same in every rank's sequence)
        ia = i - lag
        for jj in ([ia] if ia >= 0 else []):
            stall = max(0.0, svd_done[jj] - t)
            stall_total += stall
            t += stall + app + coll("bcast", 8.0 * (2 * b * b + b), P, busbw, lat)
            apply_at[jj] = t
        comm_total += comm
        exposed_total += exposed
    for jj in range(max(0, nsteps - lag), nsteps):                # drain
        stall = max(0.0, svd_done[jj] - t)
        stall_total += stall
        t += stall + max(s["apply"] for s in (r["steps"][jj] for r in runs)) + \
            coll("bcast", 8.0 * (2 * b * b + b), P, busbw, lat)
    compute = max(r["compute_s"] for r in runs)
    return {"P": P, "t_s": t / 1e3, "compute_max_rank_s": compute, "comm_s": comm_total / 1e3,
            "exposed_comm_s": exposed_total / 1e3, "svd_stall_s": stall_total / 1e3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("replay")
    ap.add_argument("--busbw", type=float, default=600.0, help="assumed NCCL bus bandwidth, GB/s")
    ap.add_argument("--lat-us", type=float, default=25.0)
    ap.add_argument("--lag", type=int, default=8)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    d = json.load(open(a.replay))
    res = {"inputs": {"replay": a.replay, "busbw_GBps_assumed": a.busbw, "latency_us": a.lat_us, "svd_lag": a.lag,
                      "svd_ms_measured": d["svd_ms"], "m": d["m"], "n": d["n"], "b": d["b"], "q": d["q"]},
           "rows": []}
    t1 = None
    for P in sorted({r["P"] for r in d["runs"]}):
        lag = a.lag if P > 1 else 1
        r = model(d, P, a.busbw, a.lat_us, lag)
        r0 = model(d, P, a.busbw, a.lat_us, 1, overlap=False)
        if P == 1:
            t1 = r["t_s"]
        r["efficiency"] = t1 / (P * r["t_s"]) if t1 else None
        r["no_overlap_lag1_t_s"] = r0["t_s"]
        r["no_overlap_lag1_efficiency"] = t1 / (P * r0["t_s"]) if t1 else None
        res["rows"].append(r)
        print(f"P={P}: t={r['t_s']:.2f} s  eff={r['efficiency']:.3f}  (compute max-rank {r['compute_max_rank_s']:.2f} s, "
              f"exposed comm {r['exposed_comm_s']:.2f} s of {r['comm_s']:.2f}, SVD stall {r['svd_stall_s']:.2f} s; "
              f"no overlap + lag 1: {r0['t_s']:.2f} s, eff {r['no_overlap_lag1_efficiency']:.3f})")
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
