"""NVLink bytes of one P2P qubit swap between 2 GPUs, from the driver's NVLink data counters
(`nvidia-smi nvlink -gt d`, KiB per link; ncu cannot profile a two-rank collective).
Expected per GPU and direction: 16 * 2^(l-1) bytes (half of the 2^l-amplitude shard).
  python tools/nvlink_bytes.py [n_local]      (2 GPUs)"""
import ctypes as C
import json
import os
import re
import subprocess
import sys
import threading

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.join(os.path.dirname(__file__), "..")))
import paper_2509_04955_b200 as pkg  # noqa: E402


def counters(dev):
    out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(dev)], capture_output=True, text=True).stdout
    tx = rx = 0
    for m in re.finditer(r"Link \d+: Data Tx: (\d+) KiB", out):
        tx += int(m.group(1))
    for m in re.finditer(r"Link \d+: Data Rx: (\d+) KiB", out):
        rx += int(m.group(1))
    return tx * 1024, rx * 1024, out


def main():
    l = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    n = l + 1
    c = pkg.Circuit.empty(n).add("h", [0])  # any circuit: the swap is driven directly below
    cid = pkg.Engine.comm_unique_id()
    engines = [None, None]

    def make(r):
        engines[r] = pkg.Engine(c, pkg.PlanOptions(), device=r, rank=r, nranks=2, comm_id=cid)

    def each(fn):
        th = [threading.Thread(target=fn, args=(r,)) for r in range(2)]
        [t.start() for t in th]
        [t.join() for t in th]

    each(make)
    L = pkg.load_qsv()
    Q = pkg.load_qsim()

    def swap(r):
        st = C.c_void_p(Q.qsim_engine_qsv_state(engines[r]._h))
        rc = L.qsv_swap(st, n - 1, l - 2, 24, 2)
        assert rc == 0, L.qsv_last_error()
        engines[r].sync()

    each(swap)  # warm: peer mapping
    before = [counters(d)[:2] for d in range(2)]
    each(swap)
    after = [counters(d)[:2] for d in range(2)]
    expect = 16 * (1 << (l - 1))
    res = {"n_local": l, "expected_bytes_per_direction": expect,
           "gpu": [{"tx": a[0] - b[0], "rx": a[1] - b[1]} for a, b in zip(after, before)]}
    for g in res["gpu"]:
        g["tx_over_expected"] = g["tx"] / expect
        g["rx_over_expected"] = g["rx"] / expect
    print(json.dumps(res))
    if before[0] == after[0]:
        print("counters did not move:", counters(0)[2][:800])
    for e in engines:
        e.close()


if __name__ == "__main__":
    main()
