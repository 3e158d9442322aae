"""Dirty-tail refresh (SURVEY §0 finding 3): the reference's reuse credit
covers a partially-filled tail block whose host image goes stale once decode
appends KV; plan_swap_out re-sends exactly that block as `refresh_ops`,
without touching the reference's counters or decisions."""

from paper_2411_18424_b200.cpu_store import CpuStore, TransferOp


def ext(blocks, start=0):
    return [(start, blocks)]


def test_partial_tail_is_refreshed_on_next_swap_out():
    st = CpuStore(1000)
    p1 = st.plan_swap_out(1, 3, ext(3, 100), tokens=40)  # block 2 holds 8 of 16 tokens
    assert p1.refresh_ops == [] and p1.moved_blocks == 3
    p2 = st.plan_swap_out(1, 4, ext(4, 100), tokens=60)  # decode filled block 2, opened 3
    assert (p2.moved_blocks, p2.reused_blocks) == (1, 3)  # reference accounting intact
    seg = st.copy_of(1).segments[0]
    host_start = st.pool.group(seg.group_id).start
    assert p2.refresh_ops == [TransferOp(1, 102, host_start + 2)]
    assert p2.all_ops() == p2.ops + p2.refresh_ops
    assert st.refreshed_blocks == 1


def test_full_tail_needs_no_refresh():
    st = CpuStore(1000)
    st.plan_swap_out(1, 3, ext(3), tokens=48)  # exactly 3 full blocks
    p = st.plan_swap_out(1, 5, ext(5), tokens=70)
    assert p.refresh_ops == []


def test_no_new_tokens_no_refresh():
    st = CpuStore(1000)
    st.plan_swap_out(1, 3, ext(3), tokens=40)
    p = st.plan_swap_out(1, 3, ext(3), tokens=40)
    assert p.moved_blocks == 0 and p.refresh_ops == []


def test_refresh_can_be_disabled_and_tokens_are_optional():
    st = CpuStore(1000)
    st.refresh_dirty_tail = False
    st.plan_swap_out(1, 3, ext(3), tokens=40)
    assert st.plan_swap_out(1, 4, ext(4), tokens=60).refresh_ops == []
    plain = CpuStore(1000)
    plain.plan_swap_out(1, 3, ext(3))
    assert plain.plan_swap_out(1, 4, ext(4)).refresh_ops == []  # reference call shape


def test_contaminated_tail_is_moved_not_refreshed():
    st = CpuStore(200)
    st.set_rank(1, 9)
    st.plan_swap_out(1, 3, ext(3), tokens=40)
    st.evict_for(0, 3)  # a higher priority takes the whole copy
    p = st.plan_swap_out(1, 4, ext(4), tokens=60)
    assert p.moved_blocks == 4 and p.refresh_ops == []


def test_prefix_swap_in_caps_saved_tokens():
    st = CpuStore(1000)
    st.plan_swap_out(1, 2, ext(2), tokens=20)
    st.plan_swap_out(1, 5, ext(5), tokens=70)
    copy = st.copy_of(1)
    copy.segments[-1].valid = False  # contaminate the second segment
    st.pool.free_group(copy.segments[-1].group_id)
    copy.segments[-1].group_id = None
    plan, kept = st.plan_swap_in_prefix(1, ext(5))
    assert kept == len(range(copy.segments[0].block_lo, copy.segments[0].block_hi))
    assert copy.saved_tokens <= kept * 16
