"""LTL syntax trees, cost functions and the canonical text form (host glue for the hot path).

Behavioural contract follows the reference's `formula.py` (paths relative to
/root/reference/pkg/src/ltllearn/): opcodes `formula.py:13-20`, enumeration order
`formula.py:24`, cost homomorphism `formula.py:132-161`, overfit construction and its
closed-form cost `formula.py:215-250`, grammar `formula.py:253-364` and printer
`formula.py:367-406`.  The learner's answer is compared *as text* against the reference, so the
printer must agree character for character; the structure of this module is our own.
"""
from __future__ import annotations

from typing import Iterator, Sequence

OP_ATOM, OP_NOT, OP_AND, OP_OR, OP_NEXT, OP_FINALLY, OP_GLOBALLY, OP_UNTIL = range(8)

#: candidate-generation order inside one cost level (reference `formula.py:24`)
CONNECTIVE_ORDER = (OP_NOT, OP_AND, OP_OR, OP_NEXT, OP_FINALLY, OP_GLOBALLY, OP_UNTIL)
UNARY_OPS = frozenset({OP_NOT, OP_NEXT, OP_FINALLY, OP_GLOBALLY})
BINARY_OPS = frozenset({OP_AND, OP_OR, OP_UNTIL})
COMMUTATIVE_OPS = frozenset({OP_AND, OP_OR})

OP_SYMBOL = {OP_NOT: "!", OP_AND: "&", OP_OR: "|", OP_NEXT: "X", OP_FINALLY: "F", OP_GLOBALLY: "G", OP_UNTIL: "U"}
_SYMBOL_OP = {v: k for k, v in OP_SYMBOL.items()}


class Formula:
    """Immutable node.  ``op`` is the opcode, ``kids`` the ordered children, ``prop`` the
    proposition index of an atom.  The named accessors (`child`, `left`, `right`) mirror the
    attribute names of the reference's node classes."""

    __slots__ = ("op", "kids", "prop", "_hash")

    def __init__(self, op: int, kids: tuple = (), prop: int = -1):
        object.__setattr__(self, "op", op)
        object.__setattr__(self, "kids", kids)
        object.__setattr__(self, "prop", prop)
        object.__setattr__(self, "_hash", None)

    def __setattr__(self, *_):
        raise AttributeError("formulae are immutable")

    @property
    def child(self) -> "Formula":
        if self.op not in UNARY_OPS:
            raise AttributeError("child")
        return self.kids[0]

    @property
    def left(self) -> "Formula":
        if self.op not in BINARY_OPS:
            raise AttributeError("left")
        return self.kids[0]

    @property
    def right(self) -> "Formula":
        if self.op not in BINARY_OPS:
            raise AttributeError("right")
        return self.kids[1]

    def __eq__(self, other):
        if self is other:
            return True
        if not isinstance(other, Formula):
            return NotImplemented
        # iterative structural comparison (overfit trees nest thousands deep)
        stack = [(self, other)]
        while stack:
            a, b = stack.pop()
            if a is b:
                continue
            if a.op != b.op or a.prop != b.prop:
                return False
            stack.extend(zip(a.kids, b.kids))
        return True

    def __hash__(self):
        if self._hash is None:
            object.__setattr__(self, "_hash", hash(print_formula(self)))
        return self._hash

    def __repr__(self):
        return f"Formula({print_formula(self)!r})"


def Atom(prop: int) -> Formula:
    return Formula(OP_ATOM, (), int(prop))


def Not(child: Formula) -> Formula:
    return Formula(OP_NOT, (child,))


def And(left: Formula, right: Formula) -> Formula:
    return Formula(OP_AND, (left, right))


def Or(left: Formula, right: Formula) -> Formula:
    return Formula(OP_OR, (left, right))


def Next(child: Formula) -> Formula:
    return Formula(OP_NEXT, (child,))


def Finally(child: Formula) -> Formula:
    return Formula(OP_FINALLY, (child,))


def Globally(child: Formula) -> Formula:
    return Formula(OP_GLOBALLY, (child,))


def Until(left: Formula, right: Formula) -> Formula:
    return Formula(OP_UNTIL, (left, right))


def opcode_of(f: Formula) -> int:
    return f.op


def make_unary(op: int, child: Formula) -> Formula:
    if op not in UNARY_OPS:
        raise ValueError(f"opcode {op} is not unary")
    return Formula(op, (child,))


def make_binary(op: int, left: Formula, right: Formula) -> Formula:
    if op not in BINARY_OPS:
        raise ValueError(f"opcode {op} is not binary")
    return Formula(op, (left, right))


def children(f: Formula) -> tuple:
    return f.kids


def iter_nodes(f: Formula) -> Iterator[Formula]:
    todo = [f]
    while todo:
        node = todo.pop()
        yield node
        todo.extend(node.kids)


# ---------------------------------------------------------------------------------- costs


class CostHomomorphism:
    """Positive weight per node kind, summed over the tree (reference `formula.py:132-156`)."""

    __slots__ = ("weights",)

    def __init__(self, weights: Sequence[int]):
        w = tuple(int(v) for v in weights)
        if len(w) != 8:
            raise ValueError("need one weight per node kind (8)")
        if min(w) < 1:
            raise ValueError("all connective weights must be >= 1")
        object.__setattr__(self, "weights", w)

    def __setattr__(self, *_):
        raise AttributeError("immutable")

    @staticmethod
    def uniform() -> "CostHomomorphism":
        return CostHomomorphism((1,) * 8)

    def of(self, op: int) -> int:
        return self.weights[op]

    def __eq__(self, other):
        return isinstance(other, CostHomomorphism) and other.weights == self.weights

    def __hash__(self):
        return hash(self.weights)

    def __repr__(self):
        return f"CostHomomorphism({self.weights})"


UNIFORM = CostHomomorphism.uniform()


def cost(f: Formula, h: CostHomomorphism = UNIFORM) -> int:
    return sum(h.weights[node.op] for node in iter_nodes(f))


def is_nnf(f: Formula) -> bool:
    return all(n.kids[0].op == OP_ATOM for n in iter_nodes(f) if n.op == OP_NOT)


def is_until_free(f: Formula) -> bool:
    return all(n.op != OP_UNTIL for n in iter_nodes(f))


def true_formula() -> Formula:
    return Or(Atom(0), Not(Atom(0)))


def false_formula() -> Formula:
    return And(Atom(0), Not(Atom(0)))


# ---------------------------------------------------------------------------------- overfit


class EmptyPositiveSet(ValueError):
    pass


def _right_nested(op_ctor, parts):
    acc = parts[-1]
    for p in parts[-2::-1]:
        acc = op_ctor(p, acc)
    return acc


def _pin_char(char: int, n_props: int) -> Formula:
    """Conjunction fixing one position: present propositions, then absent ones negated."""
    lits = [Atom(p) for p in range(n_props) if (char >> p) & 1]
    lits += [Not(Atom(p)) for p in range(n_props) if not (char >> p) & 1]
    return _right_nested(And, lits)


def _pin_trace(trace, n_props: int) -> Formula:
    f = Not(Next(true_formula()))  # "no successor": marks the end of the trace
    for char in reversed(tuple(trace)):
        f = And(_pin_char(int(char), n_props), Next(f))
    return f


def overfit(spec, alphabet) -> Formula:
    """Disjunction of exact-match formulae, one per positive trace (reference `formula.py:215-227`)."""
    if not len(spec.pos):
        raise EmptyPositiveSet("cannot overfit an empty positive set")
    return _right_nested(Or, [_pin_trace(tr, alphabet.size) for tr in spec.pos])


def overfit_cost(spec, alphabet, h: CostHomomorphism = UNIFORM) -> int:
    """Cost of ``overfit(spec)`` in closed form (reference `formula.py:230-250`).

    A literal block over n propositions with m present ones costs
    m*atom + (n-m)*(atom+not) + (n-1)*and; every position adds one `&` and one `X`; every
    trace adds the end marker; the disjunction adds |P|-1 `|` nodes.
    """
    n_traces = spec.n_pos  # (not len(spec.pos): that would materialise 2^20 tuples)
    if not n_traces:
        raise EmptyPositiveSet("cannot overfit an empty positive set")
    n = alphabet.size
    w = h.weights
    end_marker = w[OP_NOT] + w[OP_NEXT] + (2 * w[OP_ATOM] + w[OP_NOT] + w[OP_OR])
    n_positions, n_present = spec.positive_char_census()
    per_position_fixed = n * w[OP_ATOM] + (n - 1) * w[OP_AND] + w[OP_AND] + w[OP_NEXT]
    absent = n * n_positions - n_present
    return (n_traces - 1) * w[OP_OR] + n_traces * end_marker + n_positions * per_position_fixed + absent * w[OP_NOT]


# ---------------------------------------------------------------------------------- text form


class ParseError(ValueError):
    def __init__(self, message: str, position: int):
        super().__init__(f"{message} (at position {position})")
        self.position = position


_KEYWORDS = {"X", "F", "G", "U"}
_PREFIX = {"!": OP_NOT, "X": OP_NEXT, "F": OP_FINALLY, "G": OP_GLOBALLY}
_INFIX = {"&": OP_AND, "|": OP_OR, "U": OP_UNTIL}


def _lex(text: str):
    toks = []
    i, n = 0, len(text)
    while i < n:
        ch = text[i]
        if ch.isspace():
            i += 1
        elif ch in "()!&|":
            toks.append((ch, ch, i))
            i += 1
        elif ch.isalnum() or ch == "_":
            j = i + 1
            while j < n and (text[j].isalnum() or text[j] == "_"):
                j += 1
            word = text[i:j]
            toks.append((word if word in _KEYWORDS else "name", word, i))
            i = j
        else:
            raise ParseError(f"unexpected character {ch!r}", i)
    toks.append(("end", "", n))
    return toks


def parse_formula(text: str, alphabet) -> Formula:
    """Prefix ``! X F G``; infix ``& | U`` chains are right-associative; different infix
    operators may only be mixed through parentheses (reference `formula.py:253-364`)."""
    toks = _lex(text)
    pos = 0

    def operand() -> Formula:
        nonlocal pos
        prefixes = []
        while toks[pos][0] in _PREFIX:
            prefixes.append(_PREFIX[toks[pos][0]])
            pos += 1
        kind, word, at = toks[pos]
        if kind == "(":
            pos += 1
            node = chain()
            if toks[pos][0] != ")":
                raise ParseError("expected ')'", toks[pos][2])
            pos += 1
        elif kind == "name":
            pos += 1
            prop = alphabet.index_of(word)
            if prop is None:
                raise ParseError(f"unknown proposition {word!r}", at)
            node = Atom(prop)
        else:
            raise ParseError(f"expected a formula, found {kind!r}", at)
        for op in reversed(prefixes):
            node = Formula(op, (node,))
        return node

    def chain() -> Formula:
        nonlocal pos
        items = [operand()]
        infix = None
        while toks[pos][0] in _INFIX:
            kind, _, at = toks[pos]
            if infix is None:
                infix = kind
            elif kind != infix:
                raise ParseError(f"mixed infix operators {infix!r} and {kind!r} need parentheses", at)
            pos += 1
            items.append(operand())
        if infix is None:
            return items[0]
        op = _INFIX[infix]
        return _right_nested(lambda a, b: Formula(op, (a, b)), items)

    tree = chain()
    if toks[pos][0] != "end":
        raise ParseError(f"trailing input {toks[pos][0]!r}", toks[pos][2])
    return tree


def print_formula(f: Formula, alphabet=None) -> str:
    """Canonical text (reference `formula.py:367-406`): ``!`` hugs its operand, ``X F G`` take one
    space, a binary child is parenthesised unless it is the right child of the same operator."""
    pieces: list[str] = []
    work: list = [f]  # formulas to render, or literal strings to emit
    while work:
        item = work.pop()
        if type(item) is str:
            pieces.append(item)
            continue
        op = item.op
        if op == OP_ATOM:
            pieces.append(alphabet.names[item.prop] if alphabet is not None else f"p{item.prop}")
        elif op in UNARY_OPS:
            pieces.append("!" if op == OP_NOT else OP_SYMBOL[op] + " ")
            kid = item.kids[0]
            if kid.op in BINARY_OPS:
                work.extend((")", kid))
                pieces.append("(")
            else:
                work.append(kid)
        else:
            lhs, rhs = item.kids
            tail: list = []
            if rhs.op in BINARY_OPS and rhs.op != op:
                tail = [")", rhs, "("]
            else:
                tail = [rhs]
            mid = f" {OP_SYMBOL[op]} "
            if lhs.op in BINARY_OPS:
                work.extend(tail + [mid, ")", lhs, "("])
            else:
                work.extend(tail + [mid, lhs])
    return "".join(pieces)
