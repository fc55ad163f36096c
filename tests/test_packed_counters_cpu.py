"""Exactness of the packed-counter arithmetic the lower-level search kernels rely on
(DESIGN.md section 5), checked by brute force / random counts on the CPU.

* the "some field > unit" carry test ((c & M_even) + K_even) & C_even | ((c & M_odd) + K_odd) & C_odd;
* the last-part test: the sum of the fields as one coefficient of a product with a spread
  multiplier (even and odd fields separately), exact while the keys counted so far are < 2^{2w}.

These are properties of integer arithmetic at the shapes of every leaf size the kernels
enable them for (P:117 fanouts; full nodes of lower level 1 and 2)."""
import random

import pytest


def shape(leaf):
    f1 = max(2, (35 * leaf + 55 + 99) // 100)
    f2 = max(2, (21 * leaf + 90 + 99) // 100)
    return f1, f2, f1 * leaf, f1 * leaf * f2


def masks(f, w, unit):
    me = ke = ce = mo = ko = co = 0
    fm, kadd = (1 << w) - 1, (1 << w) - 1 - unit
    for j in range(f - 1):
        if (j + 1) * w > 32:
            break
        sh = j * w
        cb = 1 << (sh + w) if (j + 1) * w < 32 else 0
        if j & 1:
            mo |= fm << sh; ko |= kadd << sh; co |= cb
        else:
            me |= fm << sh; ke |= kadd << sh; ce |= cb
    ne = no = Me = Mo = 0
    for j in range(f - 1):
        if j & 1:
            Mo |= 1 << (2 * w * no); no += 1
        else:
            Me |= 1 << (2 * w * ne); ne += 1
    tope = 2 * w * (ne - 1) if ne else 0
    topo = 2 * w * (no - 1) if no else 0
    return me, ke, ce, mo, ko, co, Me, Mo, tope, topo


def classes():
    for leaf in range(2, 19):
        f1, f2, u1, u2 = shape(leaf)
        for unit, f in ((leaf, f1), (u1, f2)):
            w = (unit + 1).bit_length()
            if (f - 1) * w <= 31:
                yield leaf, unit, f, w


@pytest.mark.parametrize("leaf,unit,f,w", list(classes()))
def test_packed_overflow_and_last_part_tests_are_exact(leaf, unit, f, w):
    me, ke, ce, mo, ko, co, Me, Mo, tope, topo = masks(f, w, unit)
    m2w = (1 << (2 * w)) - 1
    rng = random.Random(1000 * leaf + unit)
    s = f * unit
    for _ in range(400):
        k = rng.randrange(1, s + 1)  # keys counted so far
        cnt_parts = [0] * f
        for _ in range(k):
            cnt_parts[rng.randrange(f)] += 1
        c = sum(cnt_parts[j] << (j * w) for j in range(f - 1)) & 0xFFFFFFFF
        some_over = any(x > unit for x in cnt_parts[: f - 1])
        flag = (((c & me) + ke) & ce) | (((c & mo) + ko) & co)
        if not some_over:
            assert flag == 0  # a valid prefix is never rejected
            if k < (1 << (2 * w)):
                se = (((c & me) * Me) % (1 << 64) >> tope) & m2w
                so = ((((c & mo) >> w) * Mo) % (1 << 64) >> topo) & m2w
                assert se + so == sum(cnt_parts[: f - 1])
                assert (se + so < k - unit) == (cnt_parts[f - 1] > unit)
        else:
            # the first field above unit is caught (fields below 2^w - 1 are exact until a
            # field overflows its width; carries only move upward)
            if max(cnt_parts[: f - 1]) <= (1 << w) - 1:
                assert flag != 0


def part_shift(p, f, w):
    """Field position of part p (narrow p*w; wide split words, 64 = not held)."""
    if (f - 1) * w <= 32:
        return p * w if p + 1 < f else 32
    hs = 32 // w
    return 64 if p + 1 >= f else (p * w if p < hs else 32 + (p - hs) * w)


@pytest.mark.parametrize("leaf", range(19, 25))
def test_wide_counter_field_extraction_is_exact(leaf):
    """The wide (64-bit, two-word) packed counters of l >= 19 and their early-rejection test
    (fields extracted one by one, k - sum > unit for the last part): a valid prefix is never
    rejected and the test rejects exactly the prefixes with a part above unit; the final
    comparison (cnt & mask) == target holds iff every part count equals unit."""
    f1, f2, u1, u2 = shape(leaf)
    rng = random.Random(leaf)
    for unit, f in ((leaf, f1), (u1, f2)):
        w = (unit + 1).bit_length()
        if (f - 1) * w <= 32:
            continue
        fm = (1 << w) - 1
        mask = sum(fm << part_shift(j, f, w) for j in range(f - 1))
        target = sum(unit << part_shift(j, f, w) for j in range(f - 1))
        s = f * unit
        for trial in range(300):
            k = rng.randrange(1, s + 1)
            parts = [0] * f
            for _ in range(k):
                parts[rng.randrange(f)] += 1
            lo = hi = 0
            for p, c in enumerate(parts):  # increments 1 << t and 1 << (t - 32), clamped
                t = part_shift(p, f, w)
                lo = (lo + (c << t if t < 32 else 0)) & 0xFFFFFFFF
                hi = (hi + (c << (t - 32) if 32 <= t < 64 else 0)) & 0xFFFFFFFF
            cnt = (hi << 32) | lo
            vals = [(cnt >> part_shift(j, f, w)) & fm for j in range(f - 1)]
            reject = any(v > unit for v in vals) or sum(vals) + unit < k
            valid = all(c <= unit for c in parts)
            if valid:
                assert not reject and vals == parts[: f - 1]
            elif max(parts[: f - 1]) < (1 << w):  # no field overflowed its width: exact verdict
                assert reject
            if k == s:
                assert ((cnt & mask) == target) == (parts == [unit] * f)
