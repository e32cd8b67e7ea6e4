"""PCIe ceiling for the host-to-host solve: pinned H2D alone, D2H alone, and both at once on
two streams (what ps_solve_host's overlapped upload/download can reach at best).
Run on the GPU box: python tools/pcie_duplex.py [GiB per direction]"""
import json
import sys

import torch


def main():
    gib = float(sys.argv[1]) if len(sys.argv) > 1 else 8.0
    n = int(gib * (1 << 30))
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        s1.synchronize()
        s2.synchronize()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e-3

    def h2d():
        with torch.cuda.stream(s1):
            s1.wait_stream(torch.cuda.current_stream())
            d_in.copy_(h_in, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)

    def d2h():
        with torch.cuda.stream(s2):
            s2.wait_stream(torch.cuda.current_stream())
            h_out.copy_(d_out, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s2)

    def chunked(k):
        c = n // k
        def both():
            for i in range(k):
                with torch.cuda.stream(s1):
                    d_in[i * c:(i + 1) * c].copy_(h_in[i * c:(i + 1) * c], non_blocking=True)
                with torch.cuda.stream(s2):
                    h_out[i * c:(i + 1) * c].copy_(d_out[i * c:(i + 1) * c], non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
        return both

    for f in (h2d, d2h):
        f()
    res = {"gib_per_direction": gib}
    res["h2d_gbs"] = n / timed(h2d) / 1e9
    res["d2h_gbs"] = n / timed(d2h) / 1e9
    res["duplex_aggregate_gbs"] = 2 * n / timed(lambda: (h2d(), d2h())) / 1e9
    res["duplex_32_chunks_aggregate_gbs"] = 2 * n / timed(chunked(32)) / 1e9
    print(json.dumps(res))


if __name__ == "__main__":
    main()
