"""NVLink traffic from the GPU's own hardware counters (NVML field values),
for checking the executor's NVLink bytes and per-dimension rates independently
of its self-reported timings (north_star (d), SURVEY.md:549-551).

ncu cannot replay a kernel whose CTAs wait on other GPUs (each replay would
wait for peers that are not replaying), so multi-GPU NVLink bytes come from
NVML's per-link data counters instead: NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX /
_RX (KiB of user data, per link, cumulative), summed over the GPU's links.

    with NvlinkCounters(device_index) as c:
        ... run + synchronize ...
    c.tx_bytes, c.rx_bytes

    python scripts/nvml_nvlink.py          # print the counters of every GPU
"""

from __future__ import annotations

import pynvml as nv

_INIT = False


def _init():
    global _INIT
    if not _INIT:
        nv.nvmlInit()
        _INIT = True


def n_links(handle) -> int:
    n = 0
    for link in range(32):
        try:
            if nv.nvmlDeviceGetNvLinkState(handle, link) == nv.NVML_FEATURE_ENABLED:
                n += 1
        except nv.NVMLError:
            break
    return n


# (tx field, rx field, unit bytes): Blackwell exposes the per-link byte
# counters (COUNT_XMIT/RCV_BYTES); older parts the KiB throughput counters
FIELD_SETS = [("NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES", "NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES", 1),
              ("NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX", 1024)]
_WORKING = {}


def _try(h, links, fs):
    tx_f, rx_f, unit = getattr(nv, fs[0]), getattr(nv, fs[1]), fs[2]
    fields = []
    for link in range(links):
        fields.append((tx_f, link))
        fields.append((rx_f, link))
    vals = nv.nvmlDeviceGetFieldValues(h, fields)
    tx = rx = 0
    for i, v in enumerate(vals):
        if v.nvmlReturn != nv.NVML_SUCCESS:
            raise RuntimeError(f"{fs[i % 2]} link {i // 2}: NVML return {v.nvmlReturn}")
        x = int(v.value.ullVal)
        if i % 2 == 0:
            tx += x
        else:
            rx += x
    return tx * unit, rx * unit


def read(index: int):
    """(tx_bytes, rx_bytes, links, field set) summed over the GPU's active links."""
    _init()
    h = nv.nvmlDeviceGetHandleByIndex(index)
    links = n_links(h)
    errs = []
    for fs in ([_WORKING[index]] if index in _WORKING else FIELD_SETS):
        try:
            tx, rx = _try(h, links, fs)
            _WORKING[index] = fs
            return tx, rx, links, fs[0]
        except Exception as e:       # try the next field set; report all if none works
            errs.append(str(e))
    raise RuntimeError("; ".join(errs))


class NvlinkCounters:
    def __init__(self, index: int):
        self.index = index

    def __enter__(self):
        self.t0 = read(self.index)
        return self

    def __exit__(self, *a):
        t1 = read(self.index)
        self.tx_bytes = t1[0] - self.t0[0]
        self.rx_bytes = t1[1] - self.t0[1]
        self.links = t1[2]
        self.field = t1[3]


if __name__ == "__main__":
    _init()
    for i in range(nv.nvmlDeviceGetCount()):
        try:
            print(i, read(i))
        except Exception as e:      # report, do not hide: the caller decides
            print(i, "error", e)
