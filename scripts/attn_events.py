"""Debug: CTA 0's attention event timeline (a -DPBS_ATTN_EVENTS build, see attn_sm100.cu).

    PBS_B200_LIB=build/events/libpbs_b200.so python scripts/attn_events.py [N]
    python scripts/attn_events.py --analyse F

MMA warp, per step (one union entry): 0 top, 1 V ready, 2 P_0 seen, 3 QK_0 issued,
4 P_1 seen, 5 QK_1 issued, 6 commits done.  Softmax group w: S wait start / S seen.
"""
import sys

import numpy as np

from attn_trace import record


def analyse(path):
    t = np.fromfile(path, dtype=np.uint64).astype(np.int64)
    mma = t[32:32 + 8192].reshape(1024, 8)
    sm = t[32 + 8192:32 + 16384].reshape(1024, 8)
    g = np.arange(100, 1000)
    g = g[np.all(mma[g][:, [0, 1, 2, 3, 4, 5, 6]] > 0, axis=1) & (mma[g + 1, 0] > 0)]
    med = lambda x: float(np.median(x))  # noqa: E731
    mean = lambda x: float(np.mean(x))  # noqa: E731
    rows = [("V wait (top -> V ready)", mma[g, 1] - mma[g, 0]),
            ("P_0 wait + PV_0 first half (V -> P_0 seen)", mma[g, 2] - mma[g, 1]),
            ("PV_0 second half + K wait + QK_0 issue", mma[g, 3] - mma[g, 2]),
            ("P_1 wait + PV_1 first half", mma[g, 4] - mma[g, 3]),
            ("PV_1 second half + QK_1 issue", mma[g, 5] - mma[g, 4]),
            ("commits", mma[g, 6] - mma[g, 5]),
            ("loop back", mma[g + 1, 0] - mma[g, 6]),
            ("period", mma[g + 1, 0] - mma[g, 0])]
    print(f"CTA 0, {len(g)} steps (SM cycles)            median     mean")
    for name, x in rows:
        print(f"  {name:44s} {med(x):7.0f} {mean(x):8.0f}")
    sm = sm[:1023]
    b = np.arange(50, 1000)
    b = b[np.all(sm[b][:, :6] > 0, axis=1) & (sm[b + 1, 0] > 0)]
    rows = [("top -> S wait (visit, partial-block fill)", sm[b, 1] - sm[b, 0]),
            ("wait S", sm[b, 2] - sm[b, 1]),
            ("load + max (incl. masking)", sm[b, 3] - sm[b, 2]),
            ("rescale", sm[b, 4] - sm[b, 3]),
            ("exp + P store + arrivals", sm[b, 5] - sm[b, 4]),
            ("loop back", sm[b + 1, 0] - sm[b, 5]),
            ("period", sm[b + 1, 0] - sm[b, 0])]
    print(f"softmax group 0 thread 0, {len(b)} blocks    median     mean")
    for name, x in rows:
        print(f"  {name:44s} {med(x):7.0f} {mean(x):8.0f}")
    p_seen = np.sort(mma[:, 2][mma[:, 2] > 0])
    arr = sm[b, 5]
    k = np.searchsorted(p_seen, arr)
    ok = k < len(p_seen)
    print(f"  P_0 arrived -> MMA sees it                  {med(p_seen[k[ok]] - arr[ok]):7.0f}")
    qk = np.sort(mma[:, 3][mma[:, 3] > 0])
    seen = sm[b, 2]
    k = np.searchsorted(qk, seen) - 1
    ok = k >= 0
    print(f"  QK_0 issued -> S seen                       {med(seen[ok] - qk[k[ok]]):7.0f}")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--analyse":
        analyse(sys.argv[2])
    else:
        analyse(record(int(sys.argv[1]) if len(sys.argv) > 1 else 131072))
