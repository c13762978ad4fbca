"""Device-resident coupled loop (les.les_main, reference les.py:419-470):
driven by a scripted stand-in for gmcf_mini.coupling (the reference is not
installed on the GPU box), the flow after the loop must equal the CPU
oracle stepped with the same inflow sequence, bitwise, and `record` must
follow the reference's bookkeeping."""

import enum
from types import SimpleNamespace

import numpy as np
import pytest

import golden_inputs as gi

pytestmark = pytest.mark.gpu


class FakeCoupling:
    """Interval of 3 steps; a new wind profile every interval; the peer
    finishes after `fin_after` syncs."""

    WIND_PROFILE_DATA_ID = 7

    class SyncStatus(enum.Enum):
        OK = 0
        PEER_FINISHED = 1

    def __init__(self, km, fin_after=100):
        self.km = km
        self.fin_after = fin_after
        self.log = []

    def init(self, tile, model_id, peers, dt, interval):
        series = SimpleNamespace(profiles=[], can_interpolate=False, next=None, count_received=0)
        return SimpleNamespace(current_time=0, series=series, interval=interval, syncs=0)

    def sync(self, st):
        st.syncs += 1
        return self.SyncStatus.PEER_FINISHED if st.syncs > self.fin_after else self.SyncStatus.OK

    def pre_exchange(self, st, data_id):
        assert data_id == self.WIND_PROFILE_DATA_ID
        n = st.series.count_received
        u, v, w = gi.default_inflow(self.km, t_seconds=60.0 * n)
        prof = SimpleNamespace(u=u, v=v, w=w, kp=self.km)
        st.series.profiles.append(prof)
        st.series.count_received += 1
        st.series.next = prof
        st.series.can_interpolate = st.series.count_received >= 2
        return self.SyncStatus.OK

    def interpolate_profile(self, series, t):
        a, b = series.profiles[-2], series.profiles[-1]
        frac = np.float64((t % 3) / 3.0)
        lerp = lambda x, y: (x.astype(np.float64) + frac * (y.astype(np.float64) - x)).astype(np.float32)  # noqa: E731
        return SimpleNamespace(u=lerp(a.u, b.u), v=lerp(a.v, b.v), w=lerp(a.w, b.w), kp=self.km)

    def advance_step(self, st):
        self.log.append(st.current_time)
        st.current_time += 1

    def finished(self, st):
        pass

    def await_peer_fins(self, st):
        pass


@pytest.mark.parametrize("fin_after", [100, 8])
def test_les_main_matches_oracle_loop(fin_after):
    import paper_1504_02264_b200 as P
    from oracle import les_oracle as O

    st = gi.config1_state()
    g = P.Grid(32, 32, 16, st["dx1"], st["dy1"], st["dzn"])
    fs = P.FlowState.create(g, dt=st["dt"], vn=st["vn"], cs=st["cs"])
    fs.mask[...] = st["mask"]
    fake = FakeCoupling(16, fin_after=fin_after)
    rec = {}
    P.les.les_main(None, 2, fs, [1], 12, 3, record=rec, coupling_module=fake, sor_iters=20)

    # the same inflow sequence through the CPU oracle
    o = O.OState.zeros(32, 32, 16)
    o.mask[...] = st["mask"]
    fake2 = FakeCoupling(16, fin_after=fin_after)
    s2 = fake2.init(None, 2, [1], 1, 3)
    steps = 0
    for _ in range(12):
        if fake2.sync(s2) is fake2.SyncStatus.PEER_FINISHED:
            break
        t = s2.current_time
        if t % 3 == 0:
            fake2.pre_exchange(s2, fake2.WIND_PROFILE_DATA_ID)
        inflow = fake2.interpolate_profile(s2.series, t - 3) if s2.series.can_interpolate else s2.series.next
        O.step(o, inflow.u, inflow.v, inflow.w, n_iter=20)
        steps += 1
        fake2.advance_step(s2)
    assert rec["steps"] == steps == min(12, fin_after)
    assert rec["profiles_received"] == s2.series.count_received
    assert rec["first_interpolation_interval"] == (2 if steps > 3 else None)
    for n in ("u", "v", "w", "fgh", "fgh_old", "p"):
        a = np.ascontiguousarray(getattr(fs, n)).view(np.uint32)
        b = np.ascontiguousarray(getattr(o, n)).view(np.uint32)
        assert np.array_equal(a, b), n
