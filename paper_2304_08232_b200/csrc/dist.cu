// dist.cu — 3D domain decomposition of the solve over the GPUs of one box:
// process grid, per-level halo plans, halo exchange with NCCL send/recv over NVLink and the
// allreduce of the CG dot products. One process per GPU; the reference itself has no distributed
// path, so the oracle for every multi-GPU result is the single-process solve on the
// global grid: all arithmetic per row is identical (same stored entries, same global column
// order), only the three dots per iteration are combined across ranks.
//
// NCCL is bound at run time (dlopen of the libnccl.so.2 that torch already loaded), so the library
// also loads on hosts without NCCL; nothing here is needed for single-GPU runs.
#include <dlfcn.h>

#include <algorithm>
#include <cstring>

#include "common.hpp"
#include "dist.hpp"
#include "kernels.cuh"

namespace slabgpu {

	// ---------------------------------------------------------------- NCCL binding

	namespace {

		constexpr int kNcclFloat64 = 8; // ncclDataType_t, nccl.h
		constexpr int kNcclSum = 0;     // ncclRedOp_t

		struct NcclApi {
			void * handle = nullptr;
			int ( *GetUniqueId )( void * id ) = nullptr;
			int ( *CommInitRank )( void ** comm, int nranks, NcclUniqueId id, int rank ) = nullptr;
			int ( *CommDestroy )( void * comm ) = nullptr;
			int ( *Send )( const void * buf, size_t count, int dtype, int peer, void * comm, cudaStream_t st ) = nullptr;
			int ( *Recv )( void * buf, size_t count, int dtype, int peer, void * comm, cudaStream_t st ) = nullptr;
			int ( *AllReduce )( const void * send, void * recv, size_t count, int dtype, int op, void * comm,
				cudaStream_t st ) = nullptr;
			int ( *GroupStart )() = nullptr;
			int ( *GroupEnd )() = nullptr;
			const char * ( *GetErrorString )( int ) = nullptr;
		};

		NcclApi & nccl() {
			static NcclApi api;
			if( api.handle != nullptr ) {
				return api;
			}
			const char * names[] = { "libnccl.so.2", "libnccl.so" };
			for( const char * name : names ) {
				api.handle = dlopen( name, RTLD_NOW | RTLD_GLOBAL );
				if( api.handle ) {
					break;
				}
			}
			if( api.handle == nullptr ) {
				fail( SLAB_ERR_CUDA, std::string( "cannot load NCCL: " ) + dlerror() );
			}
			const auto sym = [ & ]( const char * name ) {
				void * p = dlsym( api.handle, name );
				if( p == nullptr ) {
					fail( SLAB_ERR_CUDA, std::string( "NCCL symbol missing: " ) + name );
				}
				return p;
			};
			api.GetUniqueId = reinterpret_cast< decltype( api.GetUniqueId ) >( sym( "ncclGetUniqueId" ) );
			api.CommInitRank = reinterpret_cast< decltype( api.CommInitRank ) >( sym( "ncclCommInitRank" ) );
			api.CommDestroy = reinterpret_cast< decltype( api.CommDestroy ) >( sym( "ncclCommDestroy" ) );
			api.Send = reinterpret_cast< decltype( api.Send ) >( sym( "ncclSend" ) );
			api.Recv = reinterpret_cast< decltype( api.Recv ) >( sym( "ncclRecv" ) );
			api.AllReduce = reinterpret_cast< decltype( api.AllReduce ) >( sym( "ncclAllReduce" ) );
			api.GroupStart = reinterpret_cast< decltype( api.GroupStart ) >( sym( "ncclGroupStart" ) );
			api.GroupEnd = reinterpret_cast< decltype( api.GroupEnd ) >( sym( "ncclGroupEnd" ) );
			api.GetErrorString = reinterpret_cast< decltype( api.GetErrorString ) >( sym( "ncclGetErrorString" ) );
			return api;
		}

		void nccl_check( int rc, const char * what ) {
			if( rc != 0 ) {
				fail( SLAB_ERR_CUDA, std::string( what ) + ": " + nccl().GetErrorString( rc ) );
			}
		}

	} // namespace

	void nccl_unique_id( NcclUniqueId * out ) {
		nccl_check( nccl().GetUniqueId( out ), "ncclGetUniqueId" );
	}

	// ---------------------------------------------------------------- process grid

	void dist_set_grid( slab_ctx_s * ctx, int px, int py, int pz, int rank ) {
		if( px < 1 || py < 1 || pz < 1 || rank < 0 || rank >= px * py * pz ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "process grid: need px,py,pz >= 1 and 0 <= rank < px*py*pz" );
		}
		if( ctx->dist == nullptr ) {
			ctx->dist = new DistState;
		}
		DistState * d = ctx->dist;
		d->p[ 0 ] = px;
		d->p[ 1 ] = py;
		d->p[ 2 ] = pz;
		d->nranks = px * py * pz;
		d->rank = rank;
		rank_coords( d->p, rank, d->r );
	}

	void dist_init_nccl( slab_ctx_s * ctx, const NcclUniqueId * id ) {
		if( ctx->dist == nullptr ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "set the process grid before attaching a communicator" );
		}
		if( ctx->dist->comm != nullptr ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "communicator already attached" );
		}
		nccl_check( nccl().CommInitRank( &ctx->dist->comm, ctx->dist->nranks, *id, ctx->dist->rank ), "ncclCommInitRank" );
	}

	void dist_destroy( slab_ctx_s * ctx ) {
		if( ctx->dist == nullptr ) {
			return;
		}
		if( ctx->dist->comm != nullptr ) {
			nccl().CommDestroy( ctx->dist->comm );
		}
		if( ctx->dist->comm_stream != nullptr ) {
			cudaStreamDestroy( ctx->dist->comm_stream );
			cudaEventDestroy( ctx->dist->ev_boundary );
			cudaEventDestroy( ctx->dist->ev_arrived );
		}
		delete ctx->dist;
		ctx->dist = nullptr;
	}

	Decomp level_decomp( const slab_ctx_s * ctx, uint64_t lx, uint64_t ly, uint64_t lz ) {
		if( ctx->dist == nullptr ) {
			return single_domain( lx, ly, lz );
		}
		int p[ 3 ], r[ 3 ];
		std::memcpy( p, ctx->dist->p, sizeof( p ) );
		std::memcpy( r, ctx->dist->r, sizeof( r ) );
		const int l[ 3 ] = { static_cast< int >( lx ), static_cast< int >( ly ), static_cast< int >( lz ) };
		return make_decomp( l, p, r );
	}

	uint64_t ghost_capacity( const slab_ctx_s * ctx ) {
		return ctx->dist ? ctx->dist->ghost_capacity : 0;
	}

	// ---------------------------------------------------------------- halo plan

	HaloPlan * halo_plan_create( slab_ctx_s * ctx, const Decomp & D ) {
		std::unique_ptr< HaloPlan > plan( new HaloPlan );
		plan->D = D;
		const DistState * dist = ctx->dist;
		std::vector< int32_t > all_src;
		std::vector< std::vector< int32_t > > color_src( 8 ), color_dst( 8 );
		for( int dir = 0; dir < 27; ++dir ) {
			plan->peer[ dir ] = -1;
			for( int c = 0; c < 8; ++c ) {
				plan->send_off[ dir ][ c ] = static_cast< int >( all_src.size() );
				plan->send_count[ dir ][ c ] = 0;
			}
			if( dir == 13 ) {
				continue;
			}
			const int d[ 3 ] = { dir % 3 - 1, ( dir / 3 ) % 3 - 1, dir / 9 - 1 };
			if( dist != nullptr ) {
				const int nr[ 3 ] = { dist->r[ 0 ] + d[ 0 ], dist->r[ 1 ] + d[ 1 ], dist->r[ 2 ] + d[ 2 ] };
				if( nr[ 0 ] >= 0 && nr[ 0 ] < dist->p[ 0 ] && nr[ 1 ] >= 0 && nr[ 1 ] < dist->p[ 1 ] && nr[ 2 ] >= 0
					&& nr[ 2 ] < dist->p[ 2 ] ) {
					plan->peer[ dir ] = nr[ 0 ] + dist->p[ 0 ] * ( nr[ 1 ] + dist->p[ 1 ] * nr[ 2 ] );
				}
			}
			if( plan->peer[ dir ] < 0 ) {
				continue;
			}
			for( int c = 0; c < 8; ++c ) {
				std::vector< int32_t > list;
				send_list( D, dir, c, list );
				plan->send_off[ dir ][ c ] = static_cast< int >( all_src.size() );
				plan->send_count[ dir ][ c ] = static_cast< int >( list.size() );
				for( const int32_t idx : list ) {
					color_src[ c ].push_back( idx );
					color_dst[ c ].push_back( static_cast< int32_t >( all_src.size() ) );
					all_src.push_back( idx );
				}
			}
		}
		plan->total_send = static_cast< int64_t >( all_src.size() );
		try {
			SLAB_CUDA( cudaMalloc( &plan->d_send_src, std::max< size_t >( all_src.size(), 1 ) * sizeof( int32_t ) ) );
			SLAB_CUDA( cudaMalloc( &plan->d_sendbuf, std::max< size_t >( all_src.size(), 1 ) * sizeof( double ) ) );
			upload_sync( ctx->stream, plan->d_send_src, all_src.data(), all_src.size() * sizeof( int32_t ) );
			for( int c = 0; c < 8; ++c ) {
				plan->color_count[ c ] = static_cast< int64_t >( color_src[ c ].size() );
				SLAB_CUDA( cudaMalloc( &plan->d_color_src[ c ], std::max< size_t >( color_src[ c ].size(), 1 ) * sizeof( int32_t ) ) );
				SLAB_CUDA( cudaMalloc( &plan->d_color_dst[ c ], std::max< size_t >( color_src[ c ].size(), 1 ) * sizeof( int32_t ) ) );
				upload_sync( ctx->stream, plan->d_color_src[ c ], color_src[ c ].data(), color_src[ c ].size() * sizeof( int32_t ) );
				upload_sync( ctx->stream, plan->d_color_dst[ c ], color_dst[ c ].data(), color_dst[ c ].size() * sizeof( int32_t ) );
			}
		} catch( ... ) {
			halo_plan_destroy( plan.release() );
			throw;
		}
		if( ctx->dist ) {
			ctx->dist->ghost_capacity = std::max< uint64_t >( ctx->dist->ghost_capacity, static_cast< uint64_t >( D.n_ghost ) );
		}
		return plan.release();
	}

	int g_halo_overlap = 1; // compute boundary rows first and overlap their messages with the interior rows

	void halo_plan_set_boundary( slab_ctx_s * ctx, HaloPlan * plan, const std::vector< std::vector< int32_t > > & per_color,
		int64_t npos ) {
		std::vector< int32_t > all;
		std::vector< uint8_t > flags( static_cast< size_t >( npos > 0 ? npos : 1 ), 0 );
		for( int c = 0; c < 8; ++c ) {
			plan->bnd_off[ c ] = static_cast< int64_t >( all.size() );
			if( c < static_cast< int >( per_color.size() ) ) {
				for( const int32_t pos : per_color[ c ] ) {
					all.push_back( pos );
					flags[ pos ] = 1;
				}
			}
		}
		plan->bnd_off[ 8 ] = static_cast< int64_t >( all.size() );
		SLAB_CUDA( cudaMalloc( &plan->d_bnd_pos, std::max< size_t >( all.size(), 1 ) * sizeof( int32_t ) ) );
		SLAB_CUDA( cudaMalloc( &plan->d_is_bnd, flags.size() ) );
		upload_sync( ctx->stream, plan->d_bnd_pos, all.data(), all.size() * sizeof( int32_t ) );
		upload_sync( ctx->stream, plan->d_is_bnd, flags.data(), flags.size() );
	}

	bool halo_overlap_active( const slab_ctx_s * ctx, const HaloPlan * plan ) {
		return g_halo_overlap && ctx->dist != nullptr && plan != nullptr && plan->D.n_ghost > 0 && plan->d_is_bnd != nullptr;
	}

	bool halo_has_comm( const slab_ctx_s * ctx ) {
		return ctx->dist != nullptr && ctx->dist->comm != nullptr;
	}

	cudaStream_t halo_comm_stream( slab_ctx_s * ctx ) {
		DistState * d = ctx->dist;
		if( d->comm_stream == nullptr ) {
			SLAB_CUDA( cudaStreamCreateWithFlags( &d->comm_stream, cudaStreamNonBlocking ) );
			SLAB_CUDA( cudaEventCreateWithFlags( &d->ev_boundary, cudaEventDisableTiming ) );
			SLAB_CUDA( cudaEventCreateWithFlags( &d->ev_arrived, cudaEventDisableTiming ) );
		}
		return d->comm_stream;
	}

	void halo_fork( slab_ctx_s * ctx ) {
		cudaStream_t comm = halo_comm_stream( ctx );
		SLAB_CUDA( cudaEventRecord( ctx->dist->ev_boundary, ctx->stream ) );
		SLAB_CUDA( cudaStreamWaitEvent( comm, ctx->dist->ev_boundary, 0 ) );
	}

	void halo_join( slab_ctx_s * ctx ) {
		cudaStream_t comm = halo_comm_stream( ctx );
		SLAB_CUDA( cudaEventRecord( ctx->dist->ev_arrived, comm ) );
		SLAB_CUDA( cudaStreamWaitEvent( ctx->stream, ctx->dist->ev_arrived, 0 ) );
	}

	const int32_t * halo_boundary_positions( const HaloPlan * plan, int color, int64_t * count ) {
		*count = plan->bnd_off[ color + 1 ] - plan->bnd_off[ color ];
		return plan->d_bnd_pos + plan->bnd_off[ color ];
	}

	const uint8_t * halo_boundary_flags( const HaloPlan * plan ) {
		return plan->d_is_bnd;
	}

	void halo_plan_destroy( HaloPlan * plan ) {
		if( plan == nullptr ) {
			return;
		}
		cudaFree( plan->d_bnd_pos );
		cudaFree( plan->d_is_bnd );
		cudaFree( plan->d_send_src );
		cudaFree( plan->d_sendbuf );
		for( int c = 0; c < 8; ++c ) {
			cudaFree( plan->d_color_src[ c ] );
			cudaFree( plan->d_color_dst[ c ] );
		}
		delete plan;
	}

	// pack the boundary values of v (one colour, or all) into the plan's send buffer
	void halo_pack_on( cudaStream_t st, HaloPlan * plan, slab_vec_s * v, int color ) {
		if( color < 0 ) {
			kern::halo_pack( st, plan->d_send_src, nullptr, plan->total_send, v->d, plan->d_sendbuf );
		} else {
			kern::halo_pack( st, plan->d_color_src[ color ], plan->d_color_dst[ color ], plan->color_count[ color ], v->d,
				plan->d_sendbuf );
		}
	}

	void halo_pack( slab_ctx_s * ctx, HaloPlan * plan, slab_vec_s * v, int color ) {
		halo_pack_on( ctx->stream, plan, v, color );
	}

	void halo_exchange_plan( slab_ctx_s * ctx, HaloPlan * plan, slab_vec_s * v, int color, cudaStream_t stream ) {
		cudaStream_t st = stream != nullptr ? stream : ctx->stream;
		if( plan == nullptr || ctx->dist == nullptr || ctx->dist->comm == nullptr || plan->D.n_ghost == 0 ) {
			return; // single process, or manual-exchange mode (tests drive pack/unpack themselves)
		}
		if( v->n_alloc < static_cast< uint64_t >( plan->D.n_local ) + static_cast< uint64_t >( plan->D.n_ghost ) ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "vector has no room for the ghost points of this level "
				"(create vectors after the hierarchy on a distributed context)" );
		}
		halo_pack_on( st, plan, v, color );
		NcclApi & api = nccl();
		void * comm = ctx->dist->comm;
		nccl_check( api.GroupStart(), "ncclGroupStart" );
		for( int dir = 0; dir < 27; ++dir ) {
			const int peer = plan->peer[ dir ];
			if( peer < 0 ) {
				continue;
			}
			const int c0 = color < 0 ? 0 : color;
			const int c1 = color < 0 ? 8 : color + 1;
			int send_n = 0, recv_n = 0;
			for( int c = c0; c < c1; ++c ) {
				send_n += plan->send_count[ dir ][ c ];
				recv_n += plan->D.ghost_count[ dir ][ c ];
			}
			if( send_n > 0 ) {
				nccl_check( api.Send( plan->d_sendbuf + plan->send_off[ dir ][ c0 ], static_cast< size_t >( send_n ),
					kNcclFloat64, peer, comm, st ), "ncclSend" );
			}
			if( recv_n > 0 ) {
				nccl_check( api.Recv( v->d + plan->D.n_local + plan->D.ghost_base[ dir ][ c0 ], static_cast< size_t >( recv_n ),
					kNcclFloat64, peer, comm, st ), "ncclRecv" );
			}
		}
		nccl_check( api.GroupEnd(), "ncclGroupEnd" );
		ctx->dist->exchanges += 1;
	}

	void halo_exchange( slab_level_s * L, slab_vec_s * v, int color ) {
		halo_exchange_plan( L->ctx, L->plan, v, color );
	}

	void allreduce_slots( slab_ctx_s * ctx, int slot, int count ) {
		if( ctx->dist == nullptr || ctx->dist->comm == nullptr ) {
			return;
		}
		nccl_check( nccl().AllReduce( ctx->d_scalars + slot, ctx->d_scalars + slot, static_cast< size_t >( count ), kNcclFloat64, kNcclSum,
			ctx->dist->comm, ctx->stream ), "ncclAllReduce" );
	}

	void allreduce_slot( slab_ctx_s * ctx, int slot ) {
		allreduce_slots( ctx, slot, 1 );
	}

} // namespace slabgpu
