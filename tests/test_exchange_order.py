"""Host-side properties of the chunked TP exchange schedule (exchange.py): every rank processes
every owner's chunk exactly once, its own first, and every publisher serves its peers in the order
they need its rows, so the copy that is awaited soonest is issued first."""
from paper_2111_05972_b200.exchange import NWORDS, chunk_order, publish_order


def test_chunk_and_publish_orders():
    for T in range(1, 9):
        for r in range(T):
            order = chunk_order(r, T)
            assert sorted(order) == list(range(T)) and order[0] == r
        for j in range(T):
            pub = publish_order(j, T)
            assert sorted(pub + [j]) == list(range(T))
            need_step = [chunk_order(r, T).index(j) for r in pub]  # when each receiver awaits j's rows
            assert need_step == sorted(need_step) and len(set(need_step)) == len(need_step)


def test_flag_words_fit():
    assert NWORDS >= 16 * 64  # 4 ready + 4 ack kinds x 64 peers (kind + 8 for acks)
