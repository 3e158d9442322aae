"""The swap-induced decode stall estimator (live.LiveStats.stall_model): it
controls for the batch mix (KV bytes vs weight bytes differ per iteration and
between busy and quiet phases) and reports a bootstrap 95% interval, so a
swap policy that costs nothing reads as ~0 with an interval containing 0,
and a real slowdown is recovered.  Host-only (synthetic samples)."""

import numpy as np

from paper_2411_18424_b200.live import LiveStats


def _samples(rng, n, busy_frac, slowdown, kv_bias=0.0):
    out = []
    for _ in range(n):
        busy = rng.random() < busy_frac
        # busy phases carry more KV reads (preemption-heavy mixes): the naive
        # ratio would mistake the mix for a slowdown (or a speedup)
        kv = rng.uniform(0.5e9, 4e9) * (1 + (kv_bias if busy else 0))
        w = rng.uniform(2e9, 10e9)
        ms = 0.05 + kv / 5.0e9 * 1e3 + w / 7.0e9 * 1e3  # KV reads slower per byte
        ms *= (1 + slowdown) if busy else 1.0
        ms *= 1 + rng.normal(0, 0.01)
        out.append((ms, kv, w, busy, False))
    return out


def test_no_slowdown_gives_an_interval_around_zero_despite_a_mix_shift():
    st = LiveStats()
    st.samples = _samples(np.random.default_rng(1), 3000, 0.3, 0.0, kv_bias=1.0)
    # the naive ratio (one calibrated rate for every byte) is biased by the mix
    nominal = [(kv + w) / 7.0e9 * 1e3 for _, kv, w, _, _ in st.samples]
    busy = [b for *_, b, _ in st.samples]
    ratio = (sum(m for (m, *_), b in zip(st.samples, busy) if b)
             / sum(n for n, b in zip(nominal, busy) if b)) / (
        sum(m for (m, *_), b in zip(st.samples, busy) if not b)
        / sum(n for n, b in zip(nominal, busy) if not b)) - 1
    assert abs(ratio) > 0.02
    m = st.stall_model(boot=300)
    assert abs(m["stall"]) < 0.005
    assert m["ci95"][0] <= 0.0 <= m["ci95"][1]


def test_a_real_slowdown_is_recovered_with_a_tight_interval():
    st = LiveStats()
    st.samples = _samples(np.random.default_rng(2), 3000, 0.4, 0.08, kv_bias=0.5)
    m = st.stall_model(boot=300)
    assert abs(m["stall"] - 0.08) < 0.005
    assert m["ci95"][0] > 0.06 and m["ci95"][1] < 0.10
    assert m["busy_iterations"] + m["quiet_iterations"] == 3000


def test_too_few_samples_reports_none():
    st = LiveStats()
    st.samples = _samples(np.random.default_rng(3), 10, 0.5, 0.0)
    assert st.stall_model() is None


def test_busy_means_a_transfer_overlapped_the_decode_kernel_on_the_device():
    """A decode launched while a transfer was pending, but queued behind a
    device-side wait for it, ran alone: it is quiet, not busy."""
    st = LiveStats(bytes_per_us=7000.0)
    # (ms, kv, w, host flag, layered, t0, t1) on the device timeline (ms)
    st.samples = [
        (2.0, 1e9, 1e9, True, False, 10.0, 12.0),   # after a wait: transfer ended at 10
        (2.1, 1e9, 1e9, False, False, 20.0, 22.1),  # transfer [19, 30) covers it
        (2.0, 1e9, 1e9, False, False, 29.5, 31.5),  # 25% overlap: dropped
        (2.0, 1e9, 1e9, True, False, 40.0, 42.0),   # nothing running
    ]
    st.classify_by_overlap([(5.0, 10.0), (19.0, 30.0)])
    assert [x[3] for x in st.samples] == [False, True, False]
    assert st.busy_ms == 2.1 and st.quiet_ms == 4.0
    assert st.classified == "device overlap"
