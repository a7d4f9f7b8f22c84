"""Token tables and sentence boundaries.

Mirrors the reference's text core (`/root/reference/pkg/src/specstream/text.py`)
so that the algorithm layer in this package behaves identically:

* EOS is id 0 (`text.py:19`); `.`, `?`, `!` end a sentence (`text.py:28`);
* `split_words` peels punctuation off words except a `.` between two digits
  (`text.py:35-57`);
* `Vocabulary` hands out ids in order of first appearance and can be frozen
  (`text.py:60-122`); `detokenize` glues punctuation to the previous token;
* `first_sentence` returns the span through the first terminator
  (`text.py:148-157`).

`SyntheticVocabulary` is the fixed-size table the B200 decoder uses: id 0
`<eos>`, ids 1-3 the terminators, every other id `i` spelled `w<i>`. Random
prompts are word soups over the non-special ids.
"""

from __future__ import annotations

from dataclasses import dataclass

EOS_ID = 0
EOS_SURFACE = "<eos>"
PUNCTUATION = frozenset({".", ",", "?", "!", ":", ";", '"'})
SENTENCE_TERMINATORS = frozenset({".", "?", "!"})


class VocabularyError(ValueError):
    """Unknown token id or surface form."""


def _is_split_point(word: str, i: int) -> bool:
    ch = word[i]
    if ch not in PUNCTUATION:
        return False
    if ch != ".":
        return True
    inner = 0 < i < len(word) - 1
    return not (inner and word[i - 1].isdigit() and word[i + 1].isdigit())


def split_words(text: str) -> list[str]:
    pieces: list[str] = []
    for word in text.split():
        cuts = [i for i in range(len(word)) if _is_split_point(word, i)]
        cursor = 0
        for i in cuts:
            if i > cursor:
                pieces.append(word[cursor:i])
            pieces.append(word[i])
            cursor = i + 1
        if cursor < len(word):
            pieces.append(word[cursor:])
    return pieces


def _join(surfaces) -> str:
    out = []
    for s in surfaces:
        if out and not (len(s) == 1 and s in PUNCTUATION):
            out.append(" ")
        out.append(s)
    return "".join(out)


class Vocabulary:
    """First-appearance id table; id 0 is reserved for `<eos>`."""

    def __init__(self) -> None:
        self._ids: dict[str, int] = {EOS_SURFACE: EOS_ID}
        self._words: list[str] = [EOS_SURFACE]
        self._frozen = False

    def __len__(self) -> int:
        return len(self._words)

    @property
    def frozen(self) -> bool:
        return self._frozen

    def freeze(self) -> "Vocabulary":
        self._frozen = True
        return self

    def add(self, surface: str) -> int:
        if surface in self._ids:
            return self._ids[surface]
        if self._frozen:
            raise VocabularyError(f"unknown surface form {surface!r} in frozen vocabulary")
        self._ids[surface] = len(self._words)
        self._words.append(surface)
        return self._ids[surface]

    def id_of(self, surface: str) -> int:
        if surface not in self._ids:
            raise VocabularyError(f"unknown surface form {surface!r}")
        return self._ids[surface]

    def surface(self, token_id: int) -> str:
        if token_id < 0 or token_id >= len(self._words):
            raise VocabularyError(f"token id {token_id} outside vocabulary of size {len(self)}")
        return self._words[token_id]

    def tokenize(self, text: str) -> list[int]:
        lookup = self.id_of if self._frozen else self.add
        return [lookup(w) for w in split_words(text)]

    def detokenize(self, tokens) -> str:
        return _join(self.surface(t) for t in tokens)


def build_vocabulary(texts) -> Vocabulary:
    vocab = Vocabulary()
    for text in texts:
        vocab.tokenize(text)
    return vocab.freeze()


class SyntheticVocabulary:
    """Fixed `size`-entry table for the random-init decoder (always frozen)."""

    _SPECIAL = (EOS_SURFACE, ".", "?", "!")

    def __init__(self, size: int) -> None:
        if size <= len(self._SPECIAL):
            raise ValueError("synthetic vocabulary needs more than the special ids")
        self._size = size

    def __len__(self) -> int:
        return self._size

    frozen = True

    def freeze(self) -> "SyntheticVocabulary":
        return self

    def surface(self, token_id: int) -> str:
        if not 0 <= token_id < self._size:
            raise VocabularyError(f"token id {token_id} outside vocabulary of size {self._size}")
        if token_id < len(self._SPECIAL):
            return self._SPECIAL[token_id]
        return f"w{token_id}"

    def id_of(self, surface: str) -> int:
        if surface in self._SPECIAL:
            return self._SPECIAL.index(surface)
        if surface[:1] == "w" and surface[1:].isdigit():
            i = int(surface[1:])
            if len(self._SPECIAL) <= i < self._size and surface == f"w{i}":
                return i
        raise VocabularyError(f"unknown surface form {surface!r}")

    add = id_of

    def tokenize(self, text: str) -> list[int]:
        return [self.id_of(w) for w in split_words(text)]

    def detokenize(self, tokens) -> str:
        return _join(self.surface(t) for t in tokens)

    def word_ids(self) -> range:
        return range(len(self._SPECIAL), self._size)

    def judge_ids(self, text: str) -> list[int]:
        """Token ids for judge text (the consistency-judge template is English,
        which the synthetic table cannot spell): known surfaces keep their ids,
        any other word maps to a word id by 64-bit FNV-1a of its UTF-8 bytes.
        One id per `split_words` word, so a pass over it costs what
        `judge_cost` charges (lm.py:208-213)."""
        out = []
        for w in split_words(text):
            try:
                out.append(self.id_of(w))
            except VocabularyError:
                h = 0xCBF29CE484222325
                for b in w.encode("utf-8"):
                    h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
                out.append(len(self._SPECIAL) + h % (self._size - len(self._SPECIAL)))
        return out


@dataclass(frozen=True)
class SentenceSpan:
    start: int
    end: int
    terminator: str

    def __post_init__(self) -> None:
        if self.end <= self.start:
            raise ValueError("sentence span must be nonempty")
        if self.terminator not in SENTENCE_TERMINATORS:
            raise ValueError(f"{self.terminator!r} is not a sentence terminator")


def first_sentence(tokens, vocab) -> SentenceSpan | None:
    for i, tok in enumerate(tokens):
        s = vocab.surface(tok)
        if s in SENTENCE_TERMINATORS:
            return SentenceSpan(0, i + 1, s)
    return None


def sentence_spans(tokens, vocab) -> list[tuple[int, int]]:
    spans, start = [], 0
    for i, tok in enumerate(tokens):
        if vocab.surface(tok) in SENTENCE_TERMINATORS:
            spans.append((start, i + 1))
            start = i + 1
    if start < len(tokens):
        spans.append((start, len(tokens)))
    return spans


def strip_eos(tokens) -> list[int]:
    return [t for t in tokens if t != EOS_ID]


def terminator_mask(vocab) -> bytes:
    """One byte per id, 1 for a sentence terminator (uploaded to the device)."""
    return bytes(1 if vocab.surface(i) in SENTENCE_TERMINATORS else 0 for i in range(len(vocab)))
