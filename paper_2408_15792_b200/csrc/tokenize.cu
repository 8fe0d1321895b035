// prompt strings -> OPT token ids on the device.
//
// The id map is the one the scorer uses on the host (workload.prompt_token_ids): the
// prompt's whitespace tokens (str.split()), the first min(seq_len, 2048) of them
// (MAX_PROMPT_TOKENS, workload.py:23), each lower-cased and hashed as
//   id = 4 + crc32(salt + token) mod (vocab - 4)      (the reference's _token_hash,
//                                                        workload.py:125-126, salted)
// padded with pad_id; an empty prompt becomes the lone id 2 (OPT </s>); last_pos = the
// last token's index (0 when empty).
//
// Byte work, HBM-bound: one warp per prompt scans its bytes 32 at a time; a ballot of the
// whitespace bytes gives the token starts of each 32-byte window, their running count
// gives each start's token index, and each lane then hashes the tokens whose index is
// lane mod 32 with a table-driven CRC-32 over their bytes. ASCII only: str.split() and
// str.lower() are Unicode-aware, so a prompt with a byte >= 0x80 in or before its kept
// tokens is flagged (bad[i] = 1) and the caller raises — there is no host path behind it.
#include "common.cuh"

namespace rs {

constexpr int TK_WARPS = 4;

__device__ __forceinline__ bool tk_space(uint32_t b) {
    // the ASCII characters str.isspace() accepts: \t \n \v \f \r, \x1c-\x1f, space
    return b == 32u || (b >= 9u && b <= 13u) || (b >= 28u && b <= 31u);
}

__global__ void __launch_bounds__(TK_WARPS * 32) tokenize_kernel(const uint8_t* __restrict__ text,
                                                                 const int64_t* __restrict__ off, int32_t n,
                                                                 int32_t seq_len, int32_t max_tokens, uint32_t span,
                                                                 uint32_t salt_state, int32_t pad_id,
                                                                 int32_t* __restrict__ ids, int32_t* __restrict__ last,
                                                                 int32_t* __restrict__ bad) {
    __shared__ uint32_t crc_tab[256];
    extern __shared__ int32_t tk_starts[];  // [TK_WARPS][max_tokens]
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = (uint32_t)i;
#pragma unroll
        for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
        crc_tab[i] = c;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int32_t* starts = tk_starts + wid * max_tokens;
    const unsigned lt = (1u << lane) - 1u;
    for (int p = blockIdx.x * TK_WARPS + wid; p < n; p += gridDim.x * TK_WARPS) {
        const int64_t b0 = off[p], b1 = off[p + 1];
        int n_tok = 0;
        bool prev_space = true;  // the position before the prompt counts as whitespace
        unsigned nonascii = 0;
        for (int64_t base = b0; base < b1 && n_tok < max_tokens; base += 32) {
            const int64_t i = base + lane;
            const uint32_t c = i < b1 ? text[i] : 32u;
            const unsigned na = __ballot_sync(0xffffffffu, c >= 128u);
            const unsigned ws = __ballot_sync(0xffffffffu, tk_space(c));
            const unsigned before = (ws << 1) | (prev_space ? 1u : 0u);
            const unsigned st = ~ws & before;  // token starts in this window
            const int k = n_tok + __popc(st & lt);
            if (((st >> lane) & 1u) && k < max_tokens) starts[k] = (int32_t)(i - b0);
            // non-ASCII bytes matter only before the first start past the kept tokens
            // (everything before it is ASCII => Python's first max_tokens tokens are ours)
            const unsigned over = __ballot_sync(0xffffffffu, ((st >> lane) & 1u) && k >= max_tokens);
            nonascii |= na & (over ? (1u << (__ffs(over) - 1)) - 1u : 0xffffffffu);
            n_tok += __popc(st);
            prev_space = (ws >> 31) & 1u;
        }
        // the scan stops early once max_tokens starts are seen: bytes past the last
        // counted token are never read, as str.split()[:max] never looks at them either
        if (n_tok > max_tokens) n_tok = max_tokens;
        __syncwarp();
        const int64_t len = b1 - b0;
        for (int k = lane; k < seq_len; k += 32) {
            int32_t id = pad_id;
            if (k < n_tok) {
                uint32_t crc = salt_state;
                for (int64_t j = starts[k]; j < len; ++j) {
                    uint32_t c = text[b0 + j];
                    if (tk_space(c)) break;
                    nonascii |= c >= 128u;
                    if (c >= 65u && c <= 90u) c += 32u;  // ASCII lower()
                    crc = crc_tab[(crc ^ c) & 0xFFu] ^ (crc >> 8);
                }
                id = 4 + (int32_t)((crc ^ 0xFFFFFFFFu) % span);
            } else if (k == 0 && n_tok == 0) {
                id = 2;  // OPT </s>: the lone token of an empty prompt
            }
            ids[(int64_t)p * seq_len + k] = id;
        }
        nonascii = __any_sync(0xffffffffu, nonascii != 0);
        if (lane == 0) {
            last[p] = (n_tok > 0 ? n_tok : 1) - 1;
            bad[p] = nonascii ? 1 : 0;
        }
        __syncwarp();  // starts[] is rewritten by the next prompt
    }
}

}  // namespace rs

using namespace rs;

extern "C" int rs_tokenize(const uint8_t* text_dev, const int64_t* offsets_dev, int32_t n, int32_t seq_len,
                           int32_t vocab, int32_t pad_id, uint32_t salt_crc, int32_t* ids_dev, int32_t* last_dev,
                           int32_t* bad_dev, void* stream) {
    RS_NVTX();
    RS_CHECK_ARG(n >= 0 && seq_len >= 1 && vocab > 4, "rs_tokenize: need n >= 0, seq_len >= 1, vocab > 4");
    if (n == 0) return RS_OK;
    RS_CHECK_ARG(text_dev != nullptr && offsets_dev && ids_dev && last_dev && bad_dev, "rs_tokenize: NULL argument");
    const int max_tokens = seq_len < 2048 ? seq_len : 2048;  // MAX_PROMPT_TOKENS
    const size_t smem = (size_t)TK_WARPS * max_tokens * sizeof(int32_t);
    RS_CUDA(ensure_smem((const void*)tokenize_kernel, TK_WARPS * 2048 * (int)sizeof(int32_t)));
    const int need = (n + TK_WARPS - 1) / TK_WARPS, cap = num_sms() * 8;
    tokenize_kernel<<<need < cap ? need : cap, TK_WARPS * 32, smem, as_stream(stream)>>>(
        text_dev, offsets_dev, n, seq_len, max_tokens, (uint32_t)(vocab - 4), salt_crc ^ 0xFFFFFFFFu, pad_id, ids_dev,
        last_dev, bad_dev);
    RS_LAUNCH_CHECK();
    return RS_OK;
}
