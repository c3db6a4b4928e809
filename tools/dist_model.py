"""Performance model of the sharded engine (distributed.py: 512-column panels owned cyclically,
look-ahead, broadcasts on a communication stream) at P = 1, 2, 4, 8 for BASELINE configs 4
and 5, from single-B200 measurements.

    python tools/dist_model.py [bench.json] > profiles/r02_dist_model.txt

Inputs (measured on one B200, this round):
  * Ozaki GEMM rate: the bench's kernel-profiled config-4 eval_all (roofline.achieved /
    28 = FP64-equivalent TF/s), default 77.7;
  * the owner's per-block factor time (4 inner 128-wide steps: diagonal tile ~52 us, small
    DMMA products, the panel slicing) -- 0.40 ms, from the config-4 loglik pass
    (profiles/r01_config4_breakdown.json: 1.38 s for 128 blocks of which GEMMs ~1.3 s);
  * the owner's W_b build (6 DMMA products + one Ozaki GEMM of (N - c1) x 512 x 512 + slicing);
  * launch / event overhead per queued step: 10 us;
  * NCCL broadcast over NVSwitch: 350 GB/s algorithm bandwidth for these 10-400 MB messages
    (conservative: NVLink 5 is 900 GB/s per direction).
Per block step with look-ahead, a rank's compute stream runs its GEMM share while the next
panel is factored on its owner and broadcast; the step costs max(GEMM share, chain) where the
chain is what the next step waits for (owner's early panel update + factor + broadcast).
Efficiency = T(1) / (P x T(P))."""

import json
import sys

BLK = 512
SLICE_ROW = 7 * 512 + 4      # bytes per row of a 512-wide int8-sliced operand (+ exponent)


def model(n, P, rate_tf=77.7, t_factor=0.40e-3, bw=350e9, t_launch=10e-6, nmat=2, solve="w"):
    N = -(-(n + 1) // BLK) * BLK
    nb = N // BLK
    rate = rate_tf * 1e12
    gemm = lambda flops: flops / rate  # noqa: E731
    chol = fwd = right = 0.0
    for b in range(nb):
        c1 = (b + 1) * BLK
        rows = N - c1
        # trailing update of panels j > b: sum_j (N - c_j) x 512 x 512 x 2, split P ways
        upd = sum(2.0 * (N - j * BLK) * BLK * BLK for j in range(b + 1, nb))
        share = gemm(upd / P) + t_launch
        early = gemm(2.0 * rows * BLK * BLK) + t_launch if b + 1 < nb else 0.0
        bc = rows * SLICE_ROW / bw if P > 1 else 0.0
        chain = early + t_factor + bc
        chol += max(share, chain)
    if solve == "2s":
        ts = dfr = 0.0
        for b in range(nb):
            c0, c1 = b * BLK, (b + 1) * BLK
            rows = N - c1
            # syr2k of the panels j > b: 2 products x 2 (N - c_j) 512^2 per panel and matrix
            upd = sum(4.0 * (N - j * BLK) * BLK * BLK * nmat for j in range(b + 1, nb))
            share = gemm(upd / P) + t_launch
            # owner chain: W_b, steps (1)-(3), slicing, broadcast of S21 (+ P_b)
            own = (gemm(2.0 * rows * BLK * BLK) + 0.15e-3            # W_b
                   + 4.0 * BLK ** 3 * nmat / 20e12                  # (1) DMMA
                   + gemm(2.0 * 2.0 * rows * BLK * BLK * nmat)      # (2), (3)
                   + 2 * nmat * rows * BLK * 15.0 / 3.5e12)         # slicings
            bc = (nmat + 1) * rows * SLICE_ROW / bw if P > 1 else 0.0
            ts += max(share, own + bc)
            # deferred sweep block b: the panels j < b, rows c0..N
            dshare = gemm(2.0 * (N - c0) * BLK * c0 * nmat / P) + t_launch
            dfr += max(dshare, (N - c0) * SLICE_ROW / bw if P > 1 else 0.0)
        return {"chol_s": chol, "forward_s": dfr, "right_s": ts,
                "eval_all_s": chol + ts + dfr, "loglik_s": chol}
    for b in range(nb):
        c0 = b * BLK
        rows = N - c0
        # forward sweep block b: X[c0:, cols] = W_b X[c0:c1, cols] over all N columns
        share = gemm(2.0 * rows * BLK * N * nmat / P) + t_launch
        wblock = gemm(2.0 * rows * BLK * BLK) + 0.15e-3
        bc = rows * SLICE_ROW / bw if P > 1 else 0.0
        fwd += max(share, wblock + bc)
    for b in range(nb):
        c0 = b * BLK
        rows = N - c0
        upd = sum(2.0 * (N - j * BLK) * BLK * BLK * nmat for j in range(b, nb))
        share = gemm(upd / P) + t_launch
        early = gemm(2.0 * (N - (b + 1) * BLK) * BLK * BLK * nmat) if b + 1 < nb else 0.0
        slc = nmat * rows * BLK * 15.0 / 3.5e12  # slicing: 8 B read + 7 B written at 3.5 TB/s
        bc = nmat * rows * SLICE_ROW / bw if P > 1 else 0.0
        right += max(share, early + slc + bc)
    return {"chol_s": chol, "forward_s": fwd, "right_s": right,
            "eval_all_s": chol + fwd + right, "loglik_s": chol}


def main():
    rate = 77.7
    if len(sys.argv) > 1:
        line = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
        rate = line["roofline"]["fp64_equiv_tflops_algorithmic"]
    print(f"Ozaki GEMM rate {rate:.1f} TF/s FP64-equivalent (single B200, measured)")
    for solve in ("2s", "w"):
        for name, n, nmat in (("config4", 65536, 2), ("config5", 100000, 3)):
            base = model(n, 1, rate, nmat=nmat, solve=solve)
            # standard-count flops of the path: n^3/3 + nmat x (n^3 [2s] or 4n^3/3 [w])
            std = n ** 3 / 3.0 + nmat * (n ** 3 if solve == "2s" else 4.0 * n ** 3 / 3.0)
            print(f"\n{name} (n = {n}, {nmat} derivative blocks), solve path {solve}")
            print(" P   eval_all s   loglik s   eval_all eff   loglik eff   "
                  "FP64 TF/s/GPU (path's standard count)")
            for P in (1, 2, 4, 8):
                m = model(n, P, rate, nmat=nmat, solve=solve)
                eff = base["eval_all_s"] / (P * m["eval_all_s"])
                effl = base["loglik_s"] / (P * m["loglik_s"])
                tf = std / m["eval_all_s"] / P / 1e12
                print(f"{P:2d}   {m['eval_all_s']:9.3f}   {m['loglik_s']:8.3f}   {eff:11.3f}   "
                      f"{effl:10.3f}   {tf:8.1f}")


if __name__ == "__main__":
    main()
