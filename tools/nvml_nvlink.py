"""NVLink byte counters through NVML (no ncu: multi-rank kernels cannot be
replayed). Usage: python tools/nvml_nvlink.py [device ...] -- prints every
NVLink data/raw counter field NVML answers for, aggregate and per link."""
import sys

import pynvml as n

FIELDS = {"data_tx_kib": 138, "data_rx_kib": 139, "raw_tx_kib": 140, "raw_rx_kib": 141,
          "count_xmit_bytes": 202, "count_rcv_bytes": 204}


def read(handle, scope=None):
    out = {}
    for name, fid in FIELDS.items():
        try:
            req = [(fid, scope)] if scope is not None else [fid]
            v = n.nvmlDeviceGetFieldValues(handle, req)[0]
            if v.nvmlReturn == 0:
                out[name] = int(v.value.ullVal)
            else:
                out[name] = f"err{v.nvmlReturn}"
        except Exception as exc:  # noqa: BLE001
            out[name] = f"exc {exc}"
    return out


if __name__ == "__main__":
    n.nvmlInit()
    devs = [int(x) for x in sys.argv[1:]] or [0]
    for d in devs:
        h = n.nvmlDeviceGetHandleByIndex(d)
        print(d, "aggregate", read(h))
        print(d, "link0", read(h, 0))
        print(d, "scope_all", read(h, 0xFFFFFFFF))
