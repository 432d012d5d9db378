// dist.hpp — host-side types and pure functions of the domain decomposition (no CUDA calls):
// everything a test needs to check the halo plans on a machine without a GPU.
#pragma once

#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "decomp.hpp"

namespace slabgpu {

	struct NcclUniqueId {
		char internal[ 128 ]; // NCCL_UNIQUE_ID_BYTES, nccl.h:37
	};

	struct DistState {
		int p[ 3 ] = { 1, 1, 1 }; // process grid
		int r[ 3 ] = { 0, 0, 0 }; // this rank's coordinates, rank = rx + px*(ry + py*rz)
		int rank = 0, nranks = 1;
		void * comm = nullptr;    // ncclComm_t; null = manual-exchange mode
		uint64_t ghost_capacity = 0; // largest ghost count over the levels built so far
		uint64_t exchanges = 0;   // halo exchanges enqueued (diagnostics)
		cudaStream_t comm_stream = nullptr; // halo messages of a colour step travel here, beside the interior rows
		cudaEvent_t ev_boundary = nullptr;  // main stream: boundary rows done
		cudaEvent_t ev_arrived = nullptr;   // comm stream: ghosts of the colour arrived
	};

	struct HaloPlan {
		Decomp D;
		int peer[ 27 ];              // rank of the neighbour in each direction, -1 if none
		int send_off[ 27 ][ 8 ];     // first slot of (direction, colour) in the send buffer
		int send_count[ 27 ][ 8 ];
		int64_t total_send = 0;
		int32_t * d_send_src = nullptr;     // local index of every send slot, (direction, colour, natural) order
		double * d_sendbuf = nullptr;
		int32_t * d_color_src[ 8 ] = { nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr };
		int32_t * d_color_dst[ 8 ] = { nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr };
		int64_t color_count[ 8 ] = { 0, 0, 0, 0, 0, 0, 0, 0 };
		// boundary rows (= rows some neighbour holds a ghost copy of) as positions of the colour-major
		// row order, per colour, ascending; and a flag per position. They let a colour step compute its
		// boundary rows first and overlap their halo messages with the interior rows.
		int32_t * d_bnd_pos = nullptr;
		int64_t bnd_off[ 9 ] = { 0, 0, 0, 0, 0, 0, 0, 0, 0 };
		uint8_t * d_is_bnd = nullptr;
	};

	inline void rank_coords( const int p[ 3 ], int rank, int r[ 3 ] ) {
		r[ 0 ] = rank % p[ 0 ];
		r[ 1 ] = ( rank / p[ 0 ] ) % p[ 1 ];
		r[ 2 ] = rank / ( p[ 0 ] * p[ 1 ] );
	}

	// owned box of rank coordinates r on a level whose per-rank dims are l
	inline Decomp make_decomp( const int l[ 3 ], const int p[ 3 ], const int r[ 3 ] ) {
		Decomp D{};
		for( int a = 0; a < 3; ++a ) {
			D.l[ a ] = l[ a ];
			D.g[ a ] = l[ a ] * p[ a ];
			D.o[ a ] = l[ a ] * r[ a ];
		}
		D.n_local = l[ 0 ] * l[ 1 ] * l[ 2 ];
		int at = 0;
		for( int dir = 0; dir < 27; ++dir ) {
			const int d[ 3 ] = { dir % 3 - 1, ( dir / 3 ) % 3 - 1, dir / 9 - 1 };
			int start[ 3 ], len[ 3 ];
			bool inside = dir != 13;
			for( int a = 0; a < 3; ++a ) {
				dir_box( D.o[ a ], D.l[ a ], d[ a ], start[ a ], len[ a ] );
				inside = inside && start[ a ] >= 0 && start[ a ] + len[ a ] <= D.g[ a ];
			}
			for( int c = 0; c < 8; ++c ) {
				D.ghost_base[ dir ][ c ] = at;
				D.ghost_count[ dir ][ c ] = 0;
				if( inside ) {
					const int count = count_parity( start[ 0 ], len[ 0 ], c & 1 ) * count_parity( start[ 1 ], len[ 1 ], ( c >> 1 ) & 1 )
						* count_parity( start[ 2 ], len[ 2 ], ( c >> 2 ) & 1 );
					D.ghost_count[ dir ][ c ] = count;
					at += count;
				}
			}
		}
		D.n_ghost = at;
		return D;
	}

	inline Decomp single_domain_decomp( int nx, int ny, int nz ) {
		const int l[ 3 ] = { nx, ny, nz };
		const int p[ 3 ] = { 1, 1, 1 };
		const int r[ 3 ] = { 0, 0, 0 };
		return make_decomp( l, p, r );
	}

	// owned points this rank sends towards direction `dir`, colour c: the peer's ghost box for the
	// opposite direction, enumerated by the same rule (global colour, natural order)
	inline void send_list( const Decomp & D, int dir, int color, std::vector< int32_t > & out ) {
		const int d[ 3 ] = { dir % 3 - 1, ( dir / 3 ) % 3 - 1, dir / 9 - 1 };
		int start[ 3 ], len[ 3 ];
		for( int a = 0; a < 3; ++a ) {
			if( d[ a ] < 0 ) {
				start[ a ] = D.o[ a ];
				len[ a ] = 1;
			} else if( d[ a ] > 0 ) {
				start[ a ] = D.o[ a ] + D.l[ a ] - 1;
				len[ a ] = 1;
			} else {
				start[ a ] = D.o[ a ];
				len[ a ] = D.l[ a ];
			}
		}
		const int c[ 3 ] = { color & 1, ( color >> 1 ) & 1, ( color >> 2 ) & 1 };
		for( int Z = first_parity( start[ 2 ], c[ 2 ] ); Z < start[ 2 ] + len[ 2 ]; Z += 2 ) {
			for( int Y = first_parity( start[ 1 ], c[ 1 ] ); Y < start[ 1 ] + len[ 1 ]; Y += 2 ) {
				for( int X = first_parity( start[ 0 ], c[ 0 ] ); X < start[ 0 ] + len[ 0 ]; X += 2 ) {
					out.push_back( ( X - D.o[ 0 ] ) + D.l[ 0 ] * ( ( Y - D.o[ 1 ] ) + D.l[ 1 ] * ( Z - D.o[ 2 ] ) ) );
				}
			}
		}
	}

	// dist.cu
	void nccl_unique_id( NcclUniqueId * out );

} // namespace slabgpu

struct slab_ctx_s;
struct slab_vec_s;
namespace slabgpu {
	void dist_set_grid( slab_ctx_s * ctx, int px, int py, int pz, int rank );
	void dist_init_nccl( slab_ctx_s * ctx, const NcclUniqueId * id );
	void halo_pack( slab_ctx_s * ctx, HaloPlan * plan, slab_vec_s * v, int color );
}
