/*
 * distr_attn_profile.h — optional measurement hook for bench.py (not needed for computing).
 *
 * distr_attn_set_profile_events(ev_start, ev_attn, ev_end): arms a ONE-SHOT hook on the calling
 * thread. The next distr_attn_fwd_ex / exact_attn_fwd_ex call on this thread records, on its
 * own stream, ev_start before its first launch, ev_attn immediately before the fused attention
 * kernel and ev_end right after it, then disarms. Arguments are cudaEvent_t handles created by
 * the caller (any may be NULL = not recorded). Returns DA_OK. Lets the bench time the dominant
 * kernel with CUDA events on the stream it is launched on (task rule ④).
 */
#ifndef DISTR_ATTN_PROFILE_H
#define DISTR_ATTN_PROFILE_H
#ifdef __cplusplus
extern "C" {
#endif
int distr_attn_set_profile_events(void* ev_start, void* ev_attn, void* ev_end);

/* One-shot debug timeline: the next forward call on this thread makes CTA (0,0) of the attention
 * kernel write clock64() stamps of its pipeline events into device_buf (int64 [20][256], caller
 * owned; slot meanings in attn.cu). NULL disarms. Returns DA_OK. */
int distr_attn_set_trace(void* device_buf);
#ifdef __cplusplus
}
#endif
#endif
